"""Gripper import, grasp execution and force sensing (ref: pkg/src/srsim/robot)."""

from .urdf import UrdfJoint, UrdfLink, UrdfModel, parse_urdf, rpy_matrix
from .gripper import Gripper, top_down_pose
from .grasp import (GraspConfig, GraspOutcome, GraspPhase, GraspTrial, autograsp,
                    build_grasp_scene, control_step, lift_and_shake, phi, run_grasp_trial)
from .repair import RETRACT_MAX, RETRACT_STEP, RepairResult, repair_batch, repair_grasp

__all__ = ["UrdfJoint", "UrdfLink", "UrdfModel", "parse_urdf", "rpy_matrix", "Gripper",
           "top_down_pose", "GraspConfig", "GraspOutcome", "GraspPhase", "GraspTrial",
           "autograsp", "build_grasp_scene", "control_step", "lift_and_shake", "phi",
           "run_grasp_trial", "RETRACT_MAX", "RETRACT_STEP", "RepairResult", "repair_batch",
           "repair_grasp"]
