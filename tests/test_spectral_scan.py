"""Batched iteration-matrix scans: cisdc::spectral_radius_scan and
cisdc::spectral_radius on the GPU (csrc/analysis.cuh), against the UNMODIFIED reference
(oracle/_ref: analysis.cpp / linalg.cpp compiled from /root/reference).

The affine iteration matrices G are bit-identical (the engine's +, -, *, / in the reference's order,
no FMA); the spectral radius runs the same Householder + Francis QR steps, where the one libm call
(hypot, for a complex pair's modulus) is CUDA's rather than glibc's, so gamma is compared to 1e-13
relative.  Known answers: the reference's own spectral_radius cases (test_linalg.cpp:158-206).
"""
import numpy as np
import pytest

from paper_1801_01201_b200 import api

MISDC, MISDCQ, CISDCQ, IMEXQ = 0, 1, 2, 3


# ------------------------------------------------------------------ CPU: the reference-side checker

def test_reference_scan_adapter_known_shape(ref):
    """The adapter's scan returns the reference's point order: scheme, then nu (CISDCQ only), then r."""
    r = -np.logspace(-1, 3, 9)
    pts, G = ref.ref_spectral_radius_scan([MISDCQ, CISDCQ], [1, 2], r, want_G=True)
    assert len(pts) == 3 * r.size
    assert [(p.scheme, p.nu) for p in pts[:: r.size]] == [(MISDCQ, 1), (CISDCQ, 1), (CISDCQ, 2)]
    assert np.allclose([p.r for p in pts[: r.size]], r)
    assert all(p.ok for p in pts) and G.shape == (len(pts), 4, 4)


def test_reference_spectral_radius_known_answers(ref):
    """test_linalg.cpp:158-206 through the adapter (pins the checker)."""
    assert abs(ref.ref_spectral_radius(np.eye(4))[0] - 1.0) <= 1e-13
    assert abs(ref.ref_spectral_radius(np.array([[0.0, -1.0], [1.0, 0.0]]))[0] - 1.0) <= 1e-13
    comp = np.array([[-0.5, 6.5, -3.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    assert abs(ref.ref_spectral_radius(comp)[0] - 3.0) <= 3e-12
    assert ref.ref_spectral_radius(np.array([[np.nan, 0.0], [0.0, 1.0]]))[1] != 0


# ------------------------------------------------------------------ GPU vs reference

def _cmp(gpu_pts, ref_pts):
    assert len(gpu_pts) == len(ref_pts)
    for g, r in zip(gpu_pts, ref_pts):
        assert (g.scheme, g.M, g.nu, g.ok) == (r.scheme, r.M, r.nu, bool(r.ok)), (g, r)
        assert (g.a, g.d, g.r, g.dt) == (r.a, r.d, r.r, r.dt)
        if g.ok:
            assert abs(g.gamma - r.gamma) <= 1e-13 * max(1.0, abs(r.gamma)), (g, r.gamma)


@pytest.mark.gpu
@pytest.mark.parametrize("M", [2, 4, 7])
@pytest.mark.parametrize("conv", [0, 1])
def test_scan_vs_reference(gpu, ref, M, conv):
    """The figures' scan (log r grid 1e-2 .. 1e6, 40 per decade; d = r / 2) for every scheme, nu = 1, 2, 5:
    G bitwise, gamma to round-off, identical ok flags."""
    r = api.log_r_grid(-2.0, 6.0, 40)
    opt = api.ScanOptions(schemes=[MISDC, MISDCQ, CISDCQ, IMEXQ], nu_list=[1, 2, 5], r_grid=list(r), M=M,
                          convention=conv)
    pts, G = api.spectral_radius_scan(opt, return_matrices=True)
    rpts, rG = ref.ref_spectral_radius_scan(opt.schemes, opt.nu_list, r, M=M, convention=conv, want_G=True)
    _cmp(pts, rpts)
    ok = np.array([p.ok for p in pts])
    assert np.array_equal(G[ok], rG[ok])


@pytest.mark.gpu
def test_scan_fixed_d_and_singular_points(gpu, ref):
    """DRule::fixed with a d that makes a diffusion stage factor vanish at one node (ok = 0 there, as the
    reference records it), plus nu = 0 (affine_sweep_map rejects it: every such point ok = 0)."""
    M, dt = 2, 1.0
    t = api.make_quadrature_tables(M)
    d_sing = 1.0 / (dt * t.QtI[0, 0])  # 1 - coef * d == 0 at node 1 (MISDCQ / CISDCQ diffusion stage)
    r = [-0.5, -3.0, -40.0]
    opt = api.ScanOptions(schemes=[MISDCQ, CISDCQ, IMEXQ], nu_list=[0, 1], r_grid=r, d_rule=1, fixed_d=d_sing, M=M,
                          dt=dt)
    pts = api.spectral_radius_scan(opt)
    rpts, _ = ref.ref_spectral_radius_scan(opt.schemes, opt.nu_list, r, d_rule=1, fixed_d=d_sing, M=M, dt=dt)
    _cmp(pts, rpts)
    assert not all(p.ok for p in pts)


@pytest.mark.gpu
def test_spectral_radius_batch_known_answers_and_reference(gpu, ref):
    """test_linalg.cpp:158-206 on the GPU batch, plus 4096 random matrices of every size 1..8 against the
    reference (round-off), and the scaling property rho(cA) = |c| rho(A)."""
    cases = [np.eye(4), np.array([[0.0, -1.0], [1.0, 0.0]]),
             np.array([[-0.5, 6.5, -3.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])]
    want = [1.0, 1.0, 3.0]
    for A, w in zip(cases, want):
        rho, st = api.spectral_radius_batch(A)
        assert st[0] == 0 and abs(rho[0] - w) <= 3e-12
    rho, st = api.spectral_radius_batch(np.array([[np.nan, 0.0], [0.0, 1.0]]))
    assert st[0] == 1
    rng = np.random.default_rng(5)
    for n in range(1, 9):
        A = rng.uniform(-1.0, 1.0, (512, n, n))
        rho, st = api.spectral_radius_batch(A)
        assert np.all(st == 0)
        for i in range(0, 512, 37):
            rr, rc = ref.ref_spectral_radius(A[i])
            assert rc == 0 and abs(rho[i] - rr) <= 1e-13 * max(1.0, rr), (n, i)
        for c in (-2.0, 0.5):
            rc_, _ = api.spectral_radius_batch(c * A)
            assert np.all(np.abs(rc_ - abs(c) * rho) <= 1e-10 * (1.0 + rho))


@pytest.mark.gpu
def test_scan_errors(gpu):
    with pytest.raises(ValueError, match="empty r grid"):
        api.spectral_radius_scan(api.ScanOptions(schemes=[MISDCQ], r_grid=[]))
    with pytest.raises(ValueError, match="no schemes"):
        api.spectral_radius_scan(api.ScanOptions(schemes=[], r_grid=[-1.0]))
    with pytest.raises(ValueError):
        api.log_r_grid(0.0, 1.0, 0)
