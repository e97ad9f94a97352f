"""Input recipes: shapes, seeding, Σα = 1, and the hard-coded
post-shock states re-derived from the normal-shock (Rankine-Hugoniot) relations."""
import numpy as np

from paper_2409_10729_b200 import workloads as W


def _normal_shock(M, g=1.4):
    p = 1 + 2 * g / (g + 1) * (M * M - 1)
    r = (g + 1) * M * M / ((g - 1) * M * M + 2)
    u_over_c = M * (1 - 1 / r)
    return p, r, u_over_c


def test_post_shock_states():
    p, r, u = _normal_shock(1.46)
    assert np.allclose((p, r, u), W.M146, rtol=2e-5)
    p, r, u = _normal_shock(1.22)
    assert np.allclose((r, u * np.sqrt(1.4), p), W.M122_POST, rtol=2e-5)


def test_shapes_and_volume_fractions():
    for pb, v in ((W.c1_water_air(), None), (W.c2_shock_bubble(64, 32), None),
                  (W.c3_droplet(16), None), (W.c5_three_fluid(16), None),
                  (W.random_problem(3, (8, 7, 6), 3, "water"), None)):
        v = W.prims_for(pb)
        assert v.shape == pb.shape and v.dtype == np.float64 and v.flags.c_contiguous
        N, d = pb.n_fluids, pb.ndim
        a = v[N + d + 1:]
        assert np.all(a > 0) and np.allclose(a.sum(axis=0), 1.0, atol=1e-14)
        assert np.all(v[:N] > 0) and np.all(v[N + d] > 0)


def test_seeded_and_deterministic():
    pb = W.random_problem(2, (16, 8), 2, "gas")
    assert np.array_equal(W.random_prims(pb, 5), W.random_prims(pb, 5))
    assert not np.array_equal(W.random_prims(pb, 5), W.random_prims(pb, 6))
