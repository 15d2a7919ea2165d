/* C-ABI of the B200 IPC time-step library (libipc_b200.so).
 *
 * Drop-in boundary for the reference package's per-step path
 * (reference: /root/reference/pkg/src/srsim). The reference is pure Python,
 * so there is no foreign interface to re-bind; each entry point below
 * replaces the named reference function and is bound from Python with
 * ctypes (paper_2311_05945_b200/_native.py).
 *
 * Plain pointers and sizes only. Unless stated otherwise pointers are HOST
 * pointers; the library owns all device memory. Every call returns 0 on
 * success and a negative code on failure (message: ipc_last_error()).
 */
#ifndef IPC_B200_H
#define IPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ipc_world ipc_world;

/* Packed description of a batch of independent scenes ("environments").
 * Mirrors the reference scene data (scene.py:23 build_collision,
 * bodies.py GlobalState/SoftBody/AffineBody, constraints.py
 * KinematicConstraint) flattened over environments; per-environment ranges
 * are prefix arrays of length n_env + 1. All element indices are global. */
typedef struct {
  int32_t n_env, n_dof, n_vert, n_aff, n_tet, n_slot, n_tri, n_edge, n_cbody, n_cons;
  const int32_t *env_dof, *env_vert, *env_aff, *env_tet, *env_slot, *env_tri, *env_edge,
      *env_cbody, *env_cons;
  const uint8_t *env_pairs;      /* Scene.tables.needs_pair_search() */
  const uint8_t *env_has_ground; /* Scene.ground_y is not None */
  const double *env_ground_y, *env_gravity /* 3 per env */, *env_dhat, *env_kappa, *env_kappa0,
      *env_mu, *env_eps_v;
  const int32_t *vert_dof; /* DoF index of each soft vertex's x coordinate */
  const double *vert_mass;
  const int32_t *aff_dof;  /* first DoF of each affine body */
  const double *aff_M /* 144 */, *aff_acc /* 12: M_b^-1 f_gravity */, *aff_ortho /* stiffness*volume */;
  const int32_t *tet_dof;  /* 4 per tet: DoF index of each corner */
  const double *tet_Dminv /* 9 */, *tet_vol, *tet_mu, *tet_lam;
  const uint8_t *tet_model; /* 0 NeoHookean, 1 StVK, 2 FixedCorotated */
  const uint8_t *slot_aff;  /* contact slot kind: 1 = rides an affine body */
  const int32_t *slot_dof;  /* soft: DoF index; affine: body's first DoF */
  const double *slot_rest;  /* 3 per slot: rest position (affine lever arm) */
  const int32_t *slot_cbody;
  const int32_t *tri_v /* 3 */, *tri_cbody, *edge_v /* 2 */, *edge_cbody;
  const double *edge_len2;
  const uint8_t *cbody_rigid, *cbody_kin;
  const uint64_t *cbody_excl; /* bit j: excluded against env-local collision body j */
  const int32_t *cons_aff;    /* affine body index of each kinematic constraint */
  const double *cons_kappa0, *cons_mass;
  const double *x0, *v0; /* initial DoF state, n_dof each */
} ipc_world_desc;

/* ref solver.py:56 SolverConfig */
typedef struct {
  double h, newton_tol;
  int32_t max_newton_iters, max_line_search_halvings;
  double ccd_conservative_factor;
  int32_t friction_fixed_point_iters, al_max_outer;
} ipc_step_config;

/* ref solver.py:75 StepReport (per environment) */
typedef struct {
  int32_t newton_iters, ccd_invocations, converged, line_search_failed, al_outer, error;
  double final_grad_norm, min_dist_before, min_dist_after, kappa;
} ipc_step_report;

const char *ipc_last_error(void);
int ipc_device_count(void);

/* Upload a batch (replaces ref scene.py:143 make_scene's per-scene setup). */
int ipc_world_create(const ipc_world_desc *desc, ipc_world **out);
int ipc_world_destroy(ipc_world *w);

/* One implicit step of every environment (replaces ref solver.py:360 step).
 * cons_targets: 12 doubles per kinematic constraint (the bodies' target_q),
 * or NULL to keep the previous targets. reports: n_env entries or NULL. */
int ipc_world_step(ipc_world *w, const ipc_step_config *cfg, const double *cons_targets,
                   ipc_step_report *reports);
/* As ipc_world_step; enable (n_env bytes, or NULL = all) selects the
 * environments to advance — disabled ones keep their state untouched. */
int ipc_world_step_ex(ipc_world *w, const ipc_step_config *cfg, const double *cons_targets,
                      const uint8_t *enable, ipc_step_report *reports);

/* Device-resident command stream: n_steps rows of 12*n_cons targets
 * uploaded once; ipc_world_step_scheduled(k) steps with row k (no host
 * input). */
int ipc_world_upload_schedule(ipc_world *w, const double *targets, int n_steps);
int ipc_world_step_scheduled(ipc_world *w, const ipc_step_config *cfg, int k, const uint8_t *enable,
                             ipc_step_report *reports);

/* State transfer, host buffers (replaces GlobalState.gather/scatter). */
int ipc_world_get_state(ipc_world *w, double *x, double *v);
int ipc_world_set_state(ipc_world *w, const double *x, const double *v);
/* Device pointers of the resident state (n_dof doubles each). */
int ipc_world_state_device(ipc_world *w, double **x, double **v);
int ipc_world_get_kappa(ipc_world *w, double *kappa);
int ipc_world_set_kappa(ipc_world *w, const double *kappa);
/* Kinematic multipliers / penalties after the last step (12 + 1 per constraint). */
int ipc_world_get_constraints(ipc_world *w, double *lam, double *kappa);

/* World-frame contact force (N) on every slot at the current state
 * (replaces ref robot/sensing.py:30 slot_contact_forces). out: 3*n_slot. */
int ipc_world_slot_forces(ipc_world *w, double h, double *out);

/* Discrete candidates at the current state (ref broadphase.py:169), for
 * parity checks. which: 0 PT, 1 EE, 2 ground. Writes up to cap pairs
 * (2 ints each; ground: 1 int) of env `env`, returns the count via *n. */
int ipc_world_candidates(ipc_world *w, int env, int which, int32_t *out, int64_t cap, int64_t *n);

/* Per-env minimum contact distance at the current state, inf when no
 * candidate (ref contact.py:62 ContactStats.min_dist, :347). out: n_env. */
int ipc_world_min_distance(ipc_world *w, double *out);

/* Per-env minimum distance between two groups of collision bodies over
 * candidates within dhat (ref robot/proximity.py:245 min_group_distance);
 * group_a/group_b: n_env bitmasks over env-local collision body ids.
 * out: n_env (inf when no candidate pair joins the groups). */
int ipc_world_group_distance(ipc_world *w, const uint64_t *group_a, const uint64_t *group_b,
                             double *out);
/* Per-env lowest slot height above the ground over a group of collision
 * bodies (ref robot/proximity.py:76 min_ground_distance). */
int ipc_world_ground_distance(ipc_world *w, const uint64_t *group, double *out);
/* Per-env summed contact force (N, world frame) on groups of collision
 * bodies: groups = n_env*n_groups bitmasks, out = n_env*n_groups*3
 * (ref robot/sensing.py:52 body_contact_force / :61 finger_forces). */
int ipc_world_group_forces(ipc_world *w, double h, const uint64_t *groups, int n_groups,
                           double *out);

/* Bind the calling thread to a CUDA device (one process per GPU). */
int ipc_set_device(int device);

/* Instrumentation for the benchmark: per-kernel CUDA-event timing on the
 * world's stream (kernel ids: 0 broad-DCD, 1 broad-CCD, 2 pairs-deriv,
 * 3 pairs-value, 4 tet, 5 body, 6 ground, 7 friction, 8 energy-reduce,
 * 9 dense-solve, 10 ccd, 11 lags, 12 world-pos, 13 sensing, 14 misc;
 * 15 ids), launch counting, L2 flush and stream markers. */
int ipc_world_profile(ipc_world *w, int on, uint32_t kernel_mask);
int ipc_world_profile_read(ipc_world *w, double *ms, int64_t *count, int64_t *launches);
int ipc_world_flush_l2(ipc_world *w, int64_t bytes);
/* Cumulative counters: batched Newton iterations, line-search rounds, host
 * synchronisations, sparse-path PCG iterations, per-env Newton iterations and
 * line-search trials run inside the fused per-env kernels (out: 6). */
int ipc_world_stats(ipc_world *w, int64_t *out);
/* Advance every environment through steps [k0, k1) of the uploaded command
 * stream asynchronously: each env runs its own steps back to back in one CTA
 * (per-env step order preserved; envs never interact), so one env's long
 * contact-onset solve overlaps with the others' later steps. Same per-env
 * results as stepping k0..k1-1 with the fused schedule. Dense worlds only.
 * rep (optional): each env's report of its last step. Replaces a host loop
 * over ref solver.py:360 `step`. */
int ipc_world_run_scheduled(ipc_world *w, const ipc_step_config *cfg, int k0, int k1, ipc_step_report *rep);
/* Select the step schedule of a dense world: 1 = fused per-environment step
 * (one CTA runs a whole env step), 0 = batched launch sequence (default),
 * which hands the Newton loops of the last few active envs to per-env CTAs.
 * All schedules compute the same step; worlds whose env systems exceed
 * shared memory always use the batched sequence. */
int ipc_world_set_fused(ipc_world *w, int on);
/* Per-phase SM-cycle totals of the fused per-environment step (world, DCD
 * broad phase, terms, energy, dense solve, CCD prep, CCD broad phase, CCD,
 * line search, other); zeros unless the timers are on
 * (ipc_world_set_fused_timers, or IPC_FUSED_TIMERS=1 at creation). */
int ipc_world_fused_timers(ipc_world *w, int64_t *out, int n);
/* per-phase SM-cycle timers of the fused per-env kernels on/off (the phase
 * split of StepReport.times, ref solver.py:52 PHASES); instrumentation */
int ipc_world_set_fused_timers(ipc_world *w, int on);
/* SM clock of the current device (kHz): converts the fused timers' cycles */
int ipc_device_clock_khz(int32_t *khz);
int ipc_world_mark(ipc_world *w, int slot);
int ipc_world_elapsed(ipc_world *w, int a, int b, double *ms);
int ipc_world_sync(ipc_world *w);

/* Kernel-level entry points used by the parity tests (host buffers).
 * ipc_dist2_derivs: n stencils (12 doubles each) -> region, s, grad 12, hess 144
 *   (replaces ref geometry/distance.py:38/:125 + distgrad.py:95). kind 0 PT, 1 EE. */
int ipc_dist2_derivs(int kind, int64_t n, const double *stencils, int32_t *region, double *s,
                     double *grad, double *hess);
/* ref geometry/ccd.py:34 pair_ccd */
int ipc_ccd_pairs(int kind, int64_t n, const double *px, const double *pdx, double conservative,
                  double *alpha);
/* ref energy/spd.py:6 spd_project, dim in {6, 9, 12} */
int ipc_psd_project(int dim, int64_t n, double *mats);
/* ref energy/elastic.py:173-167: psi, PK1 (9), F-space Hessian (81) */
int ipc_elastic_eval(int model, int64_t n, const double *F, double mu, double lam, double *psi,
                     double *P, double *H9);

/* ---- penetrated-grasp repair (ref robot/repair.py, robot/proximity.py) ----
 * A batch of E repair problems, flattened with per-env prefix arrays.
 * Hand: env e owns links [env_link[e], env_link[e+1]); link l owns world
 * vertices [link_vert[l], link_vert[l+1]) of hand_v (placed at probe 0, i.e.
 * the input pose with the opened joints) and triangles [link_tri[l],
 * link_tri[l+1]) of hand_t (GLOBAL indices into hand_v). Object of env e:
 * vertices [env_obj_vert[e], ..) of obj_v, triangles [env_obj_tri[e], ..) of
 * obj_t (indices LOCAL to the env's object). Probe k translates the hand by
 * -retraction[k] * normal[e]. */
typedef struct ipc_repair_desc {
  int32_t n_env;
  const int32_t *env_link, *link_vert, *link_tri;
  const double *hand_v;
  const int32_t *hand_t;
  const int32_t *env_obj_vert, *env_obj_tri;
  const double *obj_v;
  const int32_t *obj_t;
  const double *normal;     /* [3E] world palm normal per env */
  int32_t n_probe;
  const double *retraction; /* [n_probe] probe distances (m) */
} ipc_repair_desc;

/* First probe whose placement has no crossing triangles and no containment
 * either way (ref repair.py:98-113 loop with _hand_object_overlap :49);
 * probe_index[e] = n_probe when no probe clears (unsalvageable). */
int ipc_repair_retract(const ipc_repair_desc *d, int32_t *probe_index);
/* device time (ms, CUDA events on the launching stream) of the last
 * ipc_repair_retract kernel launch; measurement hook, no reference analogue */
int ipc_repair_last_kernel_ms(double *ms);
/* ref proximity.py:235 max_penetration, batched: env e's points
 * [env_pt[e], env_pt[e+1]) of pts against its object mesh. */
int ipc_max_penetration(int32_t n_env, const int32_t *env_pt, const double *pts,
                        const int32_t *env_obj_vert, const int32_t *env_obj_tri,
                        const double *obj_v, const int32_t *obj_t, double *out);
/* ref proximity.py:183 winding_numbers */
int ipc_winding_numbers(int64_t n_pts, const double *pts, int32_t n_verts, const double *verts,
                        int32_t n_tris, const int32_t *tris, double *out);
/* ref proximity.py:163 count_mesh_intersections */
int ipc_count_mesh_intersections(int32_t nva, const double *va, int32_t nta, const int32_t *ta,
                                 int32_t nvb, const double *vb, int32_t ntb, const int32_t *tb,
                                 int64_t *count);

/* Measured fp64 (DFMA) throughput of the current device in TFLOP/s: the
 * compute roofline denominator of the fp64 kernels (MEASURED_PEAKS.json has
 * no fp64 figure). Instrumentation, no reference analogue. */
int ipc_measure_fp64_peak(int iters, double *tflops);

#ifdef __cplusplus
}
#endif
#endif /* IPC_B200_H */
