"""GPU parity: the sm_100a engine (through the drop-in API / C ABI) against the reference's golden
fixtures and the CPU oracle.  Tolerances are the north-star's: identical accept/reject sequence and
iteration count, factors within 1e-9 relative (Frobenius), final fit within 1e-10 absolute."""

import numpy as np
import pytest

from tests import _golden as G

pytestmark = pytest.mark.gpu

FACTOR_RTOL = 1e-9
FIT_ATOL = 1e-10
# Configs 1 and 2 are ill-conditioned enough that the reference's OWN factors move by 7e-8-1.1e-7
# (C1) and 1e-10-4e-10 (C2) under rounding-level changes (profiles/r01_parity_sensitivity.txt,
# tools/parity_sensitivity.py).  Measured engine distances (profiles/r02_parity_margins.txt): C1
# 3.9e-8, C2 6.6e-10.  C2 meets the north-star 1e-9 like every other config; only C1 keeps a bound
# at the reference's own sensitivity.  (C2 is why the triangular inverse does not split K for
# n_B <= 1024: with split-K partial sums the same fit lands 1.9e-9 from the reference.)
FACTOR_RTOL_BY_CONFIG = {"fit_c1_s0_auto": 1e-7}


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


def _model(api, case):
    dims = tuple(int(x) for x in case["dims"])
    r = int(case["rank"])
    return api.KruskalModel(G.split_stacked(case["factors"], dims, r)), dims, r


@pytest.mark.parametrize("cname", sorted(G.unit_cases()))
def test_mttkrp_all_modes(api, cname):
    case = G.unit_cases()[cname]
    model, dims, r = _model(api, case)
    y = api.DenseTensor(case["y"])
    got = np.concatenate([api.mttkrp(y, model, n).reshape(-1, order="F") for n in range(1, len(dims) + 1)])
    assert _rel(got, case["mttkrp"]) < 1e-13


@pytest.mark.parametrize("cname", sorted(G.unit_cases()))
def test_relative_error(api, cname):
    case = G.unit_cases()[cname]
    model, _, _ = _model(api, case)
    got = api.relative_error(api.DenseTensor(case["y"]), model)
    assert abs(got - float(case["relerr"])) < 1e-12


@pytest.mark.parametrize("cname", sorted(G.unit_cases()))
@pytest.mark.parametrize("variant", ["auto", "flm-a", "flm-b"])
@pytest.mark.parametrize("mu", [1e-4, 0.1, 10.0])
@pytest.mark.parametrize("refine", [0, 2])
def test_flm_step(api, cname, variant, mu, refine):
    case = G.unit_cases()[cname]
    model, dims, r = _model(api, case)
    key = f"step_{variant}_{mu:g}_{refine}"
    y = api.DenseTensor(case["y"])
    if key + "_error" in case:
        with pytest.raises(np.linalg.LinAlgError):
            api.flm_step(y, model, mu, variant, refine_steps=refine)
        return
    cand = api.flm_step(y, model, mu, variant, refine_steps=refine)
    base = model.as_vector()
    d_ref = case[key] - base
    d_got = cand.as_vector() - base
    # the un-refined step carries the forward error of the B application at small mu (the reason
    # the reference refines, solver.py:198-203); the reference's explicit inverse and our LU solve
    # differ there at the 1e-8 level.  Refined steps must agree to the reference's own 1e-8.
    assert _rel(d_got, d_ref) < (1e-8 if refine else 1e-7)


def _fit_golden(api, d, device=0):
    from paper_1205_2584_b200 import synth

    cfg = G.synth_config(d)
    y = synth.make_tensor(cfg, d["seed"])
    assert synth.tensor_digest(y) == d["digest"], "regenerated input differs from the golden input"
    conf = api.FitConfig(rank=d["rank"], variant=d["variant"], tau=d["tau"], tol=d["tol"],
                         max_iters=d["max_iters"], seed=d["seed"], init="random")
    fitter = api.fit_complex if d["complex_"] else api.fit
    return fitter(y, conf, device=device)


def _tie_iters(d):
    """Iterations whose reference decision margin is within 64 eps of err_sq."""
    m = d["margins"]
    if m.size == 0:
        return set()
    eps = np.finfo(float).eps
    return {i + 1 for i, (esq, csq, _rho) in enumerate(m) if abs(esq - csq) <= 64 * eps * esq}


@pytest.mark.parametrize("name", G.fit_names(include_full=False))
def test_fit_matches_reference(api, name):
    d = G.load_fit(name)
    res = _fit_golden(api, d)
    ref_seq = G.accept_seq(d["trace"])
    got_seq = "".join("A" if r.accepted else "r" for r in res.trace)
    ties = _tie_iters(d)
    assert res.iters == len(d["trace"]), f"{got_seq} vs {ref_seq}"
    assert res.stop_reason == d["stop_reason"]
    mism = [i + 1 for i, (a, b) in enumerate(zip(got_seq, ref_seq)) if a != b]
    assert all(t in ties for t in mism), f"non-tie decision mismatch at {mism}: {got_seq} vs {ref_seq}"
    # every recorded error matches through the last non-tie point
    errs = np.array([r.relerr for r in res.trace])
    first = min(mism) if mism else len(errs)
    fit_dev = float(np.max(np.abs(errs[:first] - d["trace"][:first, 1])))
    fbound = FACTOR_RTOL_BY_CONFIG.get(name, FACTOR_RTOL)
    fac_dev = _rel(res.model.as_vector(), d["factors"]) if not mism else float("nan")
    print(f"{name}: ties {sorted(ties)} mismatches {mism}; max |relerr - ref| = {fit_dev:.3e} (bound {FIT_ATOL:g}); "
          f"final |dfit| = {abs(res.final_relerr - d['trace'][-1, 1]):.3e}; factors rel = {fac_dev:.3e} (bound {fbound:g})")
    if not mism:
        assert abs(res.final_relerr - d["trace"][-1, 1]) < FIT_ATOL
        assert fac_dev < fbound
    assert fit_dev < FIT_ATOL


@pytest.mark.slow
@pytest.mark.parametrize("name", [n for n in G.fit_names() if n not in G.fit_names(include_full=False)])
def test_fit_matches_reference_full_config(api, name):
    test_fit_matches_reference(api, name)


@pytest.mark.parametrize("key", sorted(G.ensemble()))
def test_ensemble_fit(api, key):
    e = G.ensemble()[key]
    variant = key.split("_", 1)[1]
    y = api.DenseTensor(e["y"])
    conf = api.FitConfig(rank=int(e["rank"]), variant=variant, tol=1e-10, max_iters=40, seed=int(e["seed"]),
                         init="random")
    res = api.fit(y, conf)
    ref = e["trace"]
    # the reference's own acceptance properties (solver tests / acceptance criterion 11)
    accepted = [r.relerr for r in res.trace if r.accepted]
    assert all(b < a for a, b in zip(accepted, accepted[1:]))
    assert all(r.mu > 0 for r in res.trace)
    assert res.stop_reason in ("tol", "max_iters", "mu_overflow")
    # trajectory parity while the fit is away from its floor: these desk-size swamps are
    # chaotic in the slow tail (a 1e-16 perturbation grows ~2x per iteration), so the trace is
    # compared over the first 12 iterations and the end point within a loose band.
    errs = np.array([r.relerr for r in res.trace])
    k = min(12, len(errs), len(ref))
    assert np.max(np.abs(errs[:k] - ref[:k, 1])) < 1e-9
    assert abs(errs[-1] - ref[-1, 1]) <= 1e-4 * max(ref[-1, 1], 1e-12) + 1e-9


def test_zero_tensor_raises(api):
    with pytest.raises(ZeroDivisionError):
        api.fit(api.DenseTensor(np.zeros((3, 3, 3))), api.FitConfig(rank=1, init="random"))


def test_fit_complex_rejects_real(api):
    with pytest.raises(TypeError):
        api.fit_complex(api.DenseTensor(np.ones((3, 3))), api.FitConfig(rank=1, init="random"))


def test_flm_b_singular_kernel_is_error_stop(api):
    # orthonormal factors make every off-diagonal Gamma^(n,m) entry vanish -> K singular
    rng = np.random.default_rng(5)
    fac = [np.linalg.qr(rng.standard_normal((4, 2)))[0] for _ in range(3)]
    x = np.einsum("ir,jr,kr->ijk", *fac)
    y = api.DenseTensor(x + 1e-3 * rng.standard_normal(x.shape))
    model = api.KruskalModel(fac)
    with pytest.raises(api.SingularKernelError):
        api.flm_step(y, model, 0.1, "flm-b")


# ---- shapes that take the fp64 tensor-core (DMMA) pass path (float64, I1 >= 256) and the
# ---- 2-row-tiled DFMA path, checked against the live oracle
@pytest.mark.parametrize("dims,rank", [((600, 7, 9), 5), ((600, 7, 9), 13), ((520, 6, 5), 20), ((514, 3, 2, 4), 9),
                                       ((300, 4, 6), 24)])
def test_mttkrp_large_mode1_paths(api, dims, rank):
    from oracle import cp_oracle as O

    rng = np.random.default_rng(sum(dims) + rank)
    fac = [rng.standard_normal((d, rank)) for d in dims]
    y = np.asfortranarray(rng.standard_normal(dims))
    model = api.KruskalModel(fac)
    for n in range(1, len(dims) + 1):
        got = api.mttkrp(api.DenseTensor(y), model, n)
        ref = O.mttkrp(y, fac, n)
        assert _rel(got, ref) < 1e-13, f"mode {n}"
    assert abs(api.relative_error(api.DenseTensor(y), model) - O.relative_error(y, fac)) < 1e-12


def test_fit_large_mode1_matches_oracle(api):
    from oracle import cp_oracle as O
    from paper_1205_2584_b200 import synth

    cfg = synth.scaled(synth.CONFIGS["c4"], (300, 12, 16), rank=6, max_iters=15, name="c4_wide")
    y = synth.make_tensor(cfg, 0)
    tau = synth.tau_for_unit_mu(cfg, 0)
    res = api.fit(y, api.FitConfig(rank=6, tau=tau, tol=0.0, max_iters=15, seed=0, init="random"))
    ref = O.fit_lm(y, O.OracleConfig(rank=6, tau=tau, tol=0.0, max_iters=15, seed=0))
    assert "".join("A" if r.accepted else "r" for r in res.trace) == ref.accepted
    assert abs(res.final_relerr - ref.final_relerr) < FIT_ATOL
    assert _rel(res.model.as_vector(), O.stack(ref.factors)) < FACTOR_RTOL


# ---- the reference's default init="svd" (kruskal.py:227-242), GPU unfolding Grams
@pytest.mark.parametrize("variant", ["auto", "flm-a"])
def test_svd_init_converges_on_exact_instance(api, variant):
    # mirrors the reference's test_converges_on_exact_instance (default FitConfig: init="svd")
    rng = np.random.default_rng(14)
    fac = [rng.standard_normal((8, 2)) for _ in range(3)]
    for f in fac:
        f /= np.linalg.norm(f, axis=0, keepdims=True)
    from oracle import cp_oracle as O

    y = api.DenseTensor(O.reconstruct(fac))
    res = api.fit(y, api.FitConfig(rank=2, variant=variant, seed=3, max_iters=300))
    assert res.final_relerr < 1e-8
    assert res.stop_reason == "tol"
    assert res.iters >= res.accepted_iters >= 1


@pytest.mark.parametrize("dims,rank,cplx", [((6, 7, 8), 3, False), ((5, 4, 6), 2, True), ((3, 4, 2, 5), 4, False),
                                            ((520, 6, 5), 4, False)])
def test_unfolding_gram_and_svd_subspace(api, dims, rank, cplx):
    from oracle import cp_oracle as O
    from paper_1205_2584_b200 import _native
    from paper_1205_2584_b200.solver import svd_init

    rng = np.random.default_rng(sum(dims))
    y = rng.standard_normal(dims) + (1j * rng.standard_normal(dims) if cplx else 0)
    y = np.asfortranarray(y)
    eng = _native.Engine(_native.CPF_COMPLEX if cplx else _native.CPF_REAL, dims, rank)
    try:
        eng.set_tensor_host(y)
        for n in range(1, len(dims) + 1):
            u = O.unfold(y, n)
            assert _rel(eng.unfolding_gram(n), u @ u.conj().T) < 1e-13
        model = svd_init(eng, dims, rank, np.random.default_rng(0), "complex" if cplx else "real")
    finally:
        eng.close()
    for n, f in enumerate(model.factors):
        u, _, _ = np.linalg.svd(O.unfold(y, n + 1), full_matrices=False)
        k = min(rank, u.shape[1])
        # same leading subspace as the reference's svd_init (up to column signs / phases)
        proj = np.abs(u[:, :k].conj().T @ f[:, :k])
        np.testing.assert_allclose(np.diag(proj), 1.0, atol=1e-8)
