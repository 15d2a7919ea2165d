"""Oracle (oracle/proximity.py) against the reference's repair/proximity
golden vectors (tests/golden/make_golden_repair.py). CPU only."""

import numpy as np
import pytest

from oracle import proximity as P


@pytest.fixture(scope="module")
def prox(golden):
    return golden("proximity.npz")


@pytest.fixture(scope="module")
def geom(golden):
    return golden("repair_geom.npz")


def test_winding_numbers(prox):
    w = P.winding_numbers(prox["pts"], prox["sph_v"], prox["sph_t"])
    np.testing.assert_allclose(w, prox["w_sph"], rtol=0, atol=1e-12)
    w = P.winding_numbers(prox["pts"], prox["box_v"], prox["box_t"])
    np.testing.assert_allclose(w, prox["w_box"], rtol=0, atol=1e-12)


def test_surface_distance_and_penetration(prox):
    d = P.surface_distance(prox["pts"], prox["sph_v"], prox["sph_t"])
    np.testing.assert_allclose(d, prox["d_sph"], rtol=1e-12, atol=0)
    pen = P.max_penetration(prox["pts"], prox["sph_v"], prox["sph_t"])
    assert pen == pytest.approx(float(prox["pen_sph"]), rel=1e-12)


def test_crossing_counts(prox):
    for k, want in enumerate(prox["counts"]):
        ia, ib = prox[f"pair{k}_ids"]
        got = P.count_mesh_intersections(prox[f"pair{k}_a"], prox[f"mesh{ia}_t"],
                                         prox[f"pair{k}_b"], prox[f"mesh{ib}_t"])
        assert got == want, k
    assert (prox["counts"] > 0).sum() >= 4  # the fixture exercises real crossings


def test_surface_samples(prox):
    got = P.surface_samples(prox["box_v"], prox["box_t"])
    np.testing.assert_array_equal(got, prox["box_samples"])


def test_empty_inputs():
    v = np.zeros((3, 3))
    t = np.zeros((0, 3), np.int64)
    assert P.count_mesh_intersections(v, t, v, np.array([[0, 1, 2]])) == 0
    assert P.max_penetration(np.zeros((0, 3)), v, np.array([[0, 1, 2]])) == 0.0


def _scene(geom, k):
    from paper_2311_05945_b200 import data_path
    from paper_2311_05945_b200.robot import Gripper, parse_urdf

    return (Gripper(parse_urdf(data_path("pj_gripper.urdf"))), geom[f"s{k}_v"], geom[f"s{k}_t"],
            geom[f"s{k}_pose"], geom[f"s{k}_q"])


@pytest.mark.parametrize("k", list(range(0, 4)) + list(range(5, 37, 4)))
def test_retraction_matches_reference(geom, k):
    g, ov, ot, pose, q = _scene(geom, k)
    g.place(pose, q)
    pts = np.concatenate([P.surface_samples(b.world_vertices(), b.mesh.triangles, b.mesh.edges)
                          for b in g.bodies()])
    pen = P.max_penetration(pts, ov, ot)
    assert pen == pytest.approx(geom["pen_before"][k], rel=1e-12, abs=1e-15)
    cleared, r, _ = P.retract(g, pose, g.clamp_joints(q - 0.01), ov, ot)
    assert cleared == bool(geom["cleared"][k])
    assert r == geom["retraction"][k]  # identical accumulated probe distance


def test_retraction_schedule(geom):
    r, end = P.retraction_schedule()
    assert len(r) == 500 and r[0] == 0.0 and r[-1] <= P.RETRACT_MAX < end
    # the unsalvageable reference case stops at the first distance past the cap
    assert not geom["cleared"][4] and geom["retraction"][4] == end


def test_product_schedule_and_constants_match_reference():
    """The product's probe schedule (host side of ipc_repair_retract) is the
    reference's accumulated-distance loop, value for value."""
    from paper_2311_05945_b200.robot import repair as R

    assert (R.RETRACT_STEP, R.RETRACT_MAX) == (P.RETRACT_STEP, P.RETRACT_MAX)
    a, ea = R.retraction_schedule()
    b, eb = P.retraction_schedule()
    np.testing.assert_array_equal(a, b)
    assert ea == eb
