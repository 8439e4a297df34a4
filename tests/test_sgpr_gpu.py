"""SGPR + kernel MVM parity on the B200 against the fp64 oracle (SURVEY.md
§8(c) restatement of GPflow 2.3.1) and the reference's kernel-MVM goldens.
Gate: ELBO and predictive mean within 1e-4 relative (north star)."""

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import mvm as omvm
from oracle import sgpr as osgpr
import paper_2206_14148_b200 as tb
from paper_2206_14148_b200 import synthetic

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,ls,dtype", [("rbf", 1.3, np.float64), ("rbf", 0.8, np.float32),
                                           ("matern32", 0.5, np.float64),
                                           ("matern32", 0.7, np.float32)])
def test_sgpr_elbo_and_mean(kind, ls, dtype):
    X, y, Z, Xs = synthetic.sgpr_data(3000, 3, 150, seed=4, n_test=200, dtype=dtype)
    ref, w = osgpr.elbo(X, y, Z, kind, 1.2, ls, 0.05)
    mu_ref = osgpr.predict_mean(Xs, Z, w, kind, 1.2, ls)
    m = tb.SGPR(X, y, Z, kind, 1.2, ls, 0.05)
    e = m.elbo()
    assert abs(e - ref) <= 1e-4 * abs(ref), (e, ref)
    mu = m.predict_mean(Xs)
    assert rel_err(mu, mu_ref) <= 1e-4


@pytest.mark.parametrize("engine", ["f64", "f64_simt"])
def test_sgpr_statistics_exact(engine):
    X, y, Z, _ = synthetic.sgpr_data(5000, 4, 300, seed=5, dtype=np.float64)
    S, v, yy = osgpr.sufficient_stats(X, y, Z, "rbf", 1.0, [0.7, 1.1, 0.9, 1.3])
    m = tb.SGPR(X, y, Z, "rbf", 1.0, [0.7, 1.1, 0.9, 1.3], 0.01, engine=engine)
    st = m.statistics()
    assert rel_err(st.Sigma.cpu().numpy(), S) < 1e-12
    assert rel_err(st.v.cpu().numpy(), v) < 1e-12
    assert abs(st.yy - yy) <= 1e-12 * yy
    assert np.allclose(st.Sigma.cpu().numpy(), st.Sigma.cpu().numpy().T)


@pytest.mark.parametrize("N,M,d,kind,dtype", [(5000, 300, 4, "rbf", np.float64),
                                              (12000, 200, 3, "matern32", np.float32),
                                              (777, 129, 2, "rbf", np.float32)])
def test_sgpr_i8_statistics_are_the_exact_fixed_point_gram(N, M, d, kind, dtype):
    """The INT8 tensor-core engine returns exactly the Gram of the 24-bit
    fixed-point Kuf (oracle.sgpr.sufficient_stats_fixed24); tolerance covers
    fp64 level combination order and rare 1-ulp differences of exp() that
    move one q by 1.  Also within 1e-7 of the unquantised fp64 statistics.
    N=12000 streams two chunks (ragged last chunk); M=129 pads to 256."""
    X, y, Z, _ = synthetic.sgpr_data(N, d, M, seed=9, dtype=dtype)
    ls = [0.7, 1.1, 0.9, 1.3][:d]
    Sq, vq, yy = osgpr.sufficient_stats_fixed24(X, y, Z, kind, 1.3, ls)
    S, v, _ = osgpr.sufficient_stats(X, y, Z, kind, 1.3, ls)
    m = tb.SGPR(X, y, Z, kind, 1.3, ls, 0.01, engine="i8",
                memory_limit=None if N != 12000 else (N * d + N + M * d) * 4 + 60_000_000)
    st = m.statistics()
    if N == 12000:
        assert st.plan.chunk_n < N
    Sg = st.full_sigma().cpu().numpy()
    assert np.array_equal(Sg, Sg.T)
    assert rel_err(Sg, Sq) < 1e-11
    assert rel_err(st.v.cpu().numpy(), vq) < 1e-11
    assert rel_err(Sg, S) < 1e-7
    assert rel_err(st.v.cpu().numpy(), v) < 1e-7
    assert abs(st.yy - yy) <= 1e-12 * yy


@pytest.mark.parametrize("engine", ["i8", "f64"])
def test_sgpr_engines_agree_ill_conditioned(engine):
    """Matern-3/2, l = 0.5, dense inducing set (cond(Kuu) ~ 1e5+): the
    regime where fp32-class Gram schemes fail."""
    X, y, Z, Xs = synthetic.sgpr_data(20000, 3, 1500, seed=11, n_test=300, dtype=np.float32)
    ref, w = osgpr.elbo(X, y, Z, "matern32", 1.0, 0.5, 0.01)
    mu_ref = osgpr.predict_mean(Xs, Z, w, "matern32", 1.0, 0.5)
    m = tb.SGPR(X, y, Z, "matern32", 1.0, 0.5, 0.01, engine=engine)
    e = m.elbo()
    assert abs(e - ref) <= 1e-4 * abs(ref), (e, ref)
    assert rel_err(m.predict_mean(Xs), mu_ref) <= 1e-4


def test_sgpr_chunking_under_memory_limit():
    X, y, Z, _ = synthetic.sgpr_data(20000, 3, 500, seed=6, dtype=np.float32)
    ref, _ = osgpr.elbo(X, y, Z, "matern32", 1.0, 0.5, 0.02)
    resident = (20000 * 3 + 20000 + 500 * 3) * 4
    limit = resident + 8_000_000      # forces small chunks; the packed tail still fits
    p = tb.sgpr.plan(20000, 500, 3, kernel="matern32", memory_limit=limit)
    assert p.chunk_n < 20000 and p.peak_bytes <= limit
    e = tb.sgpr_elbo(X, y, Z, "matern32", 1.0, 0.5, 0.02, memory_limit=limit)
    assert abs(e - ref) <= 1e-4 * abs(ref)


def test_sgpr_budget_exceeded():
    X, y, Z, _ = synthetic.sgpr_data(1000, 3, 400, seed=7)
    with pytest.raises(tb.BudgetExceeded):
        tb.sgpr_elbo(X, y, Z, memory_limit="1MB")


def test_kernel_mvm_matches_reference_golden():
    g = golden("mvm_se.npz")
    graph = tb.build_kernel_mvm(700, tb.KernelSpec(float(g["variance"]), float(g["lengthscale"])))
    out, trace = tb.evaluate(graph, [g["x"], g["y"], g["v"]])
    assert rel_err(out.array, g["out"]) < 1e-13
    out2 = tb.se_kernel_mvm(g["x"], g["y"], g["v"], float(g["variance"]), float(g["lengthscale"]))
    assert rel_err(out2, g["out"]) < 1e-13


@pytest.mark.parametrize("kind", ["rbf", "matern32"])
def test_kernel_mvm_ard(kind):
    rng = np.random.default_rng(8)
    X = rng.standard_normal((777, 5))
    Z = rng.standard_normal((333, 5))
    w = rng.standard_normal(333)
    ls = [0.5, 1.0, 1.5, 2.0, 0.8]
    ref = omvm.kernel_mvm(X, Z, w, kind, 1.7, ls)
    out = tb.kernel_mvm(X, Z, w, kind, 1.7, ls)
    assert rel_err(out, ref) < 1e-13


@pytest.mark.parametrize("kind", ["rbf", "matern32"])
@pytest.mark.parametrize("dim,n,M", [(1, 5003, 2503), (11, 3001, 1031), (16, 257, 5)])
def test_kernel_mvm_ragged_tiles(kind, dim, n, M):
    """The fixed-dimension MVM kernels over several Z tiles with a ragged
    last tile, a ragged last row block, and M smaller than a tile: same
    result as the fp64 oracle, and deterministic."""
    rng = np.random.default_rng(dim + M)
    X = rng.standard_normal((n, dim))
    Z = rng.standard_normal((M, dim))
    w = rng.standard_normal(M)
    ls = list(np.linspace(0.7, 1.6, dim))
    ref = omvm.kernel_mvm(X, Z, w, kind, 1.3, ls)
    out = tb.kernel_mvm(X, Z, w, kind, 1.3, ls)
    assert rel_err(out, ref) < 1e-13
    assert np.array_equal(out, tb.kernel_mvm(X, Z, w, kind, 1.3, ls))


@pytest.mark.parametrize("N,M", [(9000, 300), (777, 129)])
def test_sgpr_i8_cta_pair_kernel_same_statistics(N, M, monkeypatch):
    """Opt-in CTA-pair Gram (tcgen05.mma.cta_group::2, TB_I8_PAIR=1) returns
    the same exact fixed-point statistics as the 1-SM kernel."""
    X, y, Z, _ = synthetic.sgpr_data(N, 3, M, seed=13, dtype=np.float32)
    Sq, vq, _ = osgpr.sufficient_stats_fixed24(X, y, Z, "matern32", 1.1, 0.6)
    ref = tb.SGPR(X, y, Z, "matern32", 1.1, 0.6, 0.01).statistics()
    monkeypatch.setenv("TB_I8_PAIR", "1")
    st = tb.SGPR(X, y, Z, "matern32", 1.1, 0.6, 0.01).statistics()
    assert st.plan.M_pad % 256 == 0
    Sg = st.full_sigma().cpu().numpy()
    assert rel_err(Sg, Sq) < 1e-11
    assert np.allclose(Sg, ref.full_sigma().cpu().numpy(), rtol=1e-13, atol=0)


@pytest.mark.parametrize("kind,engine,dtype", [("rbf", "f64", np.float64),
                                               ("matern32", "f64", np.float64),
                                               ("rbf", "i8", np.float32),
                                               ("matern32", "i8", np.float32)])
def test_elbo_gradient_matches_finite_differences(kind, engine, dtype):
    """GPflow-style training gradient (variance, ARD lengthscales, noise, Z)
    vs central finite differences of the fp64 oracle ELBO.  The N-streaming
    part runs through tb_sgpr_kuf_grad over several chunks."""
    X, y, Z, _ = synthetic.sgpr_data(3000, 3, 25, seed=17, dtype=dtype)
    ls = [0.9, 1.3, 0.7]
    m = tb.SGPR(X, y, Z, kind, 1.4, ls, 0.05, engine=engine)
    e, g = m.elbo_and_grads(chunk_n=1024)
    ref_e, _ = osgpr.elbo(X, y, Z, kind, 1.4, ls, 0.05)
    assert abs(e - ref_e) <= 1e-6 * abs(ref_e)
    fd = osgpr.elbo_grads_fd(X, y, Z, kind, 1.4, ls, 0.05)
    tol = 1e-5 if engine == "f64" else 1e-3
    for key in ("variance", "noise_variance", "lengthscales", "Z"):
        got, want = np.asarray(g[key], np.float64), np.asarray(fd[key], np.float64)
        assert np.max(np.abs(got - want)) <= tol * max(np.max(np.abs(want)), 1.0), (key, got, want)


def test_gradient_memory_estimate_and_budget():
    """elbo_and_grads is N-independent in memory but its dense autograd tail
    is O(M^2): grad_memory_bytes must bound torch's measured peak (and not by
    much), and a memory_limit below it raises BudgetExceeded before work."""
    import torch
    from paper_2206_14148_b200.sgpr import grad_memory_bytes
    N, d, M, chunk = 30000, 4, 1536, 2048
    X, y, Z, _ = synthetic.sgpr_data(N, d, M, seed=5, dtype=np.float32)
    m = tb.SGPR(X, y, Z, "rbf", 1.0, 0.7, 0.05, tail="dense")
    m.statistics()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    m.elbo_and_grads(chunk_n=chunk)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    est = grad_memory_bytes(M, d, chunk)
    assert peak <= est <= 2.0 * peak, (peak, est)
    resident = (X.size + y.size + Z.size) * 4
    small = tb.SGPR(X, y, Z, "rbf", 1.0, 0.7, 0.05, memory_limit=resident + est // 2,
                    tail="dense")
    with pytest.raises(tb.BudgetExceeded):
        small.elbo_and_grads(chunk_n=chunk)


@pytest.mark.parametrize("kind", ["rbf", "matern32"])
def test_packed_tail_matches_dense_tail(kind):
    """The in-place packed-tile tail (Kuu = LL^T, Kuu + Sigma/s2 = PP^T,
    X = L^-1 P) gives GPflow's ELBO and predictive mean like the dense
    cuSOLVER tail (two-sided solve), at cond(Kuu) ~ 1e5 (Matern l=0.5) and
    5e5 (RBF l=0.25).  (The fixed-point statistics hold the 1e-4 mean gate to
    cond ~ 1e7; beyond that use engine="f64".)"""
    X, y, Z, Xs = synthetic.sgpr_data(20000, 3, 1500, seed=11, n_test=300, dtype=np.float32)
    ls = 0.5 if kind == "matern32" else 0.25
    ref, w = osgpr.elbo(X, y, Z, kind, 1.0, ls, 0.01)
    mu_ref = osgpr.predict_mean(Xs, Z, w, kind, 1.0, ls)
    packed = tb.SGPR(X, y, Z, kind, 1.0, ls, 0.01, tail="packed")
    dense = tb.SGPR(X, y, Z, kind, 1.0, ls, 0.01, tail="dense")
    ep, ed = packed.elbo(), dense.elbo()
    # the ELBO is a small difference of O(N var / s2) = 2e6 terms; the two
    # formulations round those terms differently at ~1e-10 of their size
    scale = max(abs(ed), 20000 * 1.0 / 0.01)
    assert abs(ep - ed) <= 1e-9 * scale
    assert abs(ep - ref) <= 1e-4 * abs(ref)
    mp = packed.predict_mean(Xs)
    # w = (Kuu + Sigma/s2)^-1 v / s2 vs GPflow's L^-T LB^-T c: equal in exact
    # arithmetic, different fp64 rounding orders (~1e-5 apart at cond 2e8 in
    # numpy); both within the 1e-4 gate
    assert rel_err(mp, dense.predict_mean(Xs)) < 5e-5
    assert rel_err(mp, mu_ref) <= 1e-4
    e2, _ = packed.elbo_and_grads(chunk_n=4096)      # statistics recomputed after the tail
    assert abs(e2 - ed) <= 1e-9 * scale


def test_whole_elbo_evaluation_within_memory_limit():
    """Statistics AND the O(M^3) tail inside memory_limit (inputs counted, as
    the reference's budget does): the packed tail keeps two packed M x M
    matrices; the dense tail would need several full ones."""
    import torch
    X, y, Z, Xs = synthetic.sgpr_data(60000, 3, 3000, seed=12, n_test=100, dtype=np.float32)
    Xd, yd, Zd = (torch.from_numpy(a).cuda() for a in (X, y, Z))
    limit = 160 * 10**6
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated() - (Xd.numel() + yd.numel() + Zd.numel()) * 4
    torch.cuda.reset_peak_memory_stats()
    m = tb.SGPR(Xd, yd, Zd, "matern32", 1.0, 0.6, 0.02, memory_limit=limit)
    e = m.elbo()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    assert peak <= limit, (peak, limit)
    ref, _ = osgpr.elbo(X, y, Z, "matern32", 1.0, 0.6, 0.02)
    assert abs(e - ref) <= 1e-4 * abs(ref)


def test_sgpr_c4_shape_matches_golden():
    """The benchmarked SGPR configuration's shape (BASELINE.json configs[3]:
    d = 11, M = 1e4, RBF l = 1, variance 1, noise 0.01, memory_limit 1 GB)
    at N = 3e4 against tests/golden/sgpr_c4_shape.npz (fp64 oracle, made by
    tests/golden/make_sgpr_c4_golden.py).  Runs the d = 11 instance of the
    Kuf quantiser, the 79-tile Gram (ragged last 12x12 super-block) over
    several chunks, and the 79-tile packed tail.  Statistics are held to the
    exact 24-bit fixed-point Gram; ELBO and mean to the quantised oracle
    (fp64 rounding of the two tail formulations only) and to the unquantised
    one (the north-star 1e-4 gate)."""
    import hashlib
    import torch
    g = golden("sgpr_c4_shape.npz")
    N, d, M = int(g["N"]), int(g["d"]), int(g["M"])
    X, y, Z, Xs = synthetic.sgpr_data(N, d, M, seed=int(g["seed"]), n_test=300,
                                      dtype=np.float32, z="normal")
    h = hashlib.sha256()
    for a in (X, y, Z, Xs):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(g["x_sha"]), "synthetic generator drifted"
    var, ls, noise = float(g["variance"]), float(g["lengthscale"]), float(g["noise"])
    m = tb.SGPR(X, y, Z, "rbf", var, ls, noise, memory_limit="1GB", engine="i8")
    st = m.statistics()
    assert int(st.plan.M_pad) == 79 * 128
    assert int(st.plan.chunk_n) < N                      # several chunks, ragged last
    assert rel_err(st.v.cpu().numpy(), g["v_q"]) < 1e-11
    assert abs(st.yy - float(g["yy"])) <= 1e-12 * float(g["yy"])
    S = st.full_sigma()
    assert rel_err(S.diagonal().cpu().numpy(), g["diag_q"]) < 1e-11
    assert rel_err(S[torch.from_numpy(g["rows"]).cuda()].cpu().numpy(), g["rows_q"]) < 1e-11
    r = torch.from_numpy(np.random.default_rng(7).standard_normal(M)).cuda()
    assert rel_err((S @ r).cpu().numpy(), g["check_q"]) < 1e-11
    del S
    e = m.elbo()
    scale = N * var / noise                              # size of the cancelling terms
    assert abs(e - float(g["elbo_q"])) <= 1e-9 * scale, (e, float(g["elbo_q"]))
    assert abs(e - float(g["elbo"])) <= 1e-4 * abs(float(g["elbo"]))
    mu = m.predict_mean(Xs)
    assert rel_err(mu, g["mean_q"]) < 1e-8
    assert rel_err(mu, g["mean"]) <= 1e-4


def test_sgpr_full_c4_i8_engine_matches_fp64_engine():
    """Full C4 (N = 2e6, d = 11, M = 1e4, RBF, as bench.py generates it):
    the default fixed-point INT8 engine + packed tail (inside 1 GB) against
    the fp64 DMMA engine + dense cuSOLVER tail on the same data."""
    import torch
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(77)
    X = torch.randn((2_000_000, 11), generator=gen, device=dev)
    y = (torch.sin(X.double().sum(1)) + 0.1 * torch.randn(X.shape[0], generator=gen, device=dev,
                                                          dtype=torch.float64)).float()
    gen.manual_seed(5)
    Z = torch.randn((10_000, 11), generator=gen, device=dev)
    Xs = torch.randn((300, 11), generator=gen, device=dev)
    a = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit="1GB", engine="i8")
    ea = a.elbo()
    mua = a.predict_mean(Xs)
    b = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, engine="f64", tail="dense")
    eb = b.elbo()
    mub = b.predict_mean(Xs)
    mua, mub = (t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t) for t in (mua, mub))
    assert abs(ea - eb) <= 1e-6 * abs(eb), (ea, eb)
    assert rel_err(mua, mub) <= 1e-4


@pytest.mark.parametrize("N,d,M,kind", [(3000, 3, 25, "rbf"), (5000, 3, 300, "matern32"),
                                        (4000, 11, 200, "rbf")])
def test_packed_gradient_matches_finite_differences_and_dense(N, d, M, kind):
    """The in-budget gradient (tb_sgpr_grad_run: packed factors, column
    panels, fused data kernel) against central differences of the fp64
    oracle ELBO and against the dense autograd-free path on the same
    fixed-point statistics; M = 300 pads to 3 tiles, d = 11 takes the
    16-wide instance of the data kernel."""
    X, y, Z, _ = synthetic.sgpr_data(N, d, M, seed=17, dtype=np.float32)
    ls = [0.9, 1.3, 0.7, 1.1, 0.8, 1.2, 1.0, 0.95, 1.05, 1.15, 0.85][:d]
    e1, g1 = tb.SGPR(X, y, Z, kind, 1.4, ls, 0.05).elbo_and_grads()
    e2, g2 = tb.SGPR(X, y, Z, kind, 1.4, ls, 0.05, tail="dense").elbo_and_grads(chunk_n=1024)
    assert abs(e1 - e2) <= 1e-9 * abs(e2)
    for key in ("variance", "noise_variance", "lengthscales", "Z"):
        a, b = np.asarray(g1[key], np.float64), np.asarray(g2[key], np.float64)
        assert np.max(np.abs(a - b)) <= 1e-6 * max(np.max(np.abs(b)), 1.0), key
    if M <= 25:
        fd = osgpr.elbo_grads_fd(X, y, Z, kind, 1.4, ls, 0.05)
        for key in ("variance", "noise_variance", "lengthscales", "Z"):
            a, b = np.asarray(g1[key], np.float64), np.asarray(fd[key], np.float64)
            assert np.max(np.abs(a - b)) <= 1e-3 * max(np.max(np.abs(b)), 1.0), key


def test_packed_gradient_inside_memory_limit():
    """elbo_and_grads at a limit the dense tail cannot meet: the packed path
    plans its peak (grad_peak_bytes), stays under the limit on the device
    and returns the dense path's numbers."""
    import torch
    N, d, M = 30000, 3, 1500
    X, y, Z, _ = synthetic.sgpr_data(N, d, M, seed=19, dtype=np.float32)
    from paper_2206_14148_b200.sgpr import grad_memory_bytes
    resident = (N * d + N + M * d) * 4
    limit = resident + 2 * 8 * M * M // 2 + 24 * 10**6     # ~ two packed triangles + panels
    assert grad_memory_bytes(M, d) + resident > limit          # the dense tail would not fit
    Xd, yd, Zd = (torch.from_numpy(a).cuda() for a in (X, y, Z))
    m = tb.SGPR(Xd, yd, Zd, "matern32", 1.0, 0.6, 0.02, memory_limit=limit)
    planned = m.grad_peak_bytes()
    assert planned <= limit
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated() - (Xd.numel() + yd.numel() + Zd.numel()) * 4
    torch.cuda.reset_peak_memory_stats()
    e, g = m.elbo_and_grads()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    assert peak <= limit, (peak, limit)
    e2, g2 = tb.SGPR(X, y, Z, "matern32", 1.0, 0.6, 0.02, tail="dense").elbo_and_grads()
    assert abs(e - e2) <= 1e-9 * abs(e2)
    # Matern l = 0.6 with 1500 inducing points is ill-conditioned (cond(Kuu)
    # ~ 1e5+): the two tails' explicit-inverse vs triangular-solve rounding
    # differ at ~1e-5 of the largest dELBO/dZ entry
    for key in ("variance", "noise_variance", "lengthscales", "Z"):
        a, b = np.asarray(g[key], np.float64), np.asarray(g2[key], np.float64)
        assert np.max(np.abs(a - b)) <= 1e-4 * max(np.max(np.abs(b)), 1.0), key


def test_packed_tail_falls_back_when_A_is_too_ill_conditioned():
    """cond(Kuu + Sigma/s2) ~ 1e14 (2-D inputs, long lengthscales, dense
    inducing points, jitter 1e-6): the packed in-place factorisation of A
    meets a negative pivot, so the ELBO and the gradient take GPflow's dense
    formulation (Cholesky of B = I + L^-1 Sigma L^-T / s2) - same answer as
    the fp64 oracle, no error."""
    X, y, Z, Xs = synthetic.sgpr_data(15364, 2, 432, seed=70, n_test=64, dtype=np.float32)
    var, ls, noise = 1.8588339123918893, [2.4, 1.35], 0.05396516393244166
    ref, w = osgpr.elbo(X, y, Z, "rbf", var, ls, noise)
    m = tb.SGPR(X, y, Z, "rbf", var, ls, noise)
    e = m.elbo()
    assert abs(e - ref) <= 1e-4 * abs(ref)
    assert rel_err(m.predict_mean(Xs), osgpr.predict_mean(Xs, Z, w, "rbf", var, ls)) <= 1e-4
    e2, g = tb.SGPR(X, y, Z, "rbf", var, ls, noise).elbo_and_grads()
    assert abs(e2 - ref) <= 1e-4 * abs(ref)
    assert np.all(np.isfinite(np.asarray(g["Z"])))
