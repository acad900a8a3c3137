"""GPU: the speculative rejection branch (engine.cu plan_spec) against the oracle.

The branch factors Phi(Grams_t, mu_t * growth_t) -- the core system a rho <= 0 rejection needs next
-- beside the candidate.  A rejection with rho > 0 and cand_err >= err (solver.py:358-361: mu SHRINKS,
growth resets) must not take it.  That case needs a negative gain-ratio denominator, which the
goldens never hit, so a test hook (CPF_TEST_NEGDENOM=t in the engine, OracleConfig.negate_denom_at in
the oracle) negates the denominator at iteration t of a step the reference rejected with rho < 0:
the same step then has rho > 0 and is still rejected.  Both branch settings (CPF_SPEC=0/1) must
follow the oracle's trajectory and be bitwise identical to each other."""

import numpy as np
import pytest

from tests import _golden as G
from tests.test_gpu_parity import FACTOR_RTOL, FIT_ATOL, _rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


# (golden, iteration the reference rejected with rho < 0)
CASES = [("fit_c0_s0_auto", 8), ("fit_c0_s0_auto", 11), ("fit_c3_mini_s0_auto", 7)]


def _fit(api, monkeypatch, d, spec, t):
    from paper_1205_2584_b200 import synth

    monkeypatch.setenv("CPF_SPEC", str(spec))
    monkeypatch.setenv("CPF_TEST_NEGDENOM", str(t))
    y = synth.make_tensor(G.synth_config(d), d["seed"])
    conf = api.FitConfig(rank=d["rank"], variant=d["variant"], tau=d["tau"], tol=d["tol"],
                         max_iters=d["max_iters"], seed=d["seed"], init="random")
    return (api.fit_complex if d["complex_"] else api.fit)(y, conf), y


@pytest.mark.parametrize("name,t", CASES)
def test_rho_positive_rejection_matches_oracle(api, monkeypatch, name, t):
    from oracle import cp_oracle as O

    d = G.load_fit(name)
    assert d["trace"][t - 1, 3] == 0 and d["margins"][t - 1, 2] < 0, "case must be a rho < 0 rejection"
    res0, y = _fit(api, monkeypatch, d, 0, t)
    res1, _ = _fit(api, monkeypatch, d, 1, t)
    ref = O.fit_lm(y, O.OracleConfig(rank=d["rank"], variant=d["variant"], tau=d["tau"], tol=d["tol"],
                                     max_iters=d["max_iters"], seed=d["seed"], negate_denom_at=t))
    # the hooked step is a rho > 0 rejection: mu shrank although the step was rejected
    assert ref.trace[t - 1][3] is False and ref.trace[t - 1][2] < ref.trace[t - 2][2]
    eps = np.finfo(float).eps
    ties = {i + 1 for i, (esq, csq, _rho) in enumerate(ref.detail) if abs(esq - csq) <= 64 * eps * esq}
    ref_errs = np.array([e for (_, e, _, _) in ref.trace])
    for res in (res0, res1):
        seq = "".join("A" if r.accepted else "r" for r in res.trace)
        mism = [i + 1 for i, (a, b) in enumerate(zip(seq, ref.accepted)) if a != b]
        assert all(i in ties for i in mism), f"non-tie decision mismatch at {mism}: {seq} vs {ref.accepted}"
        errs = np.array([r.relerr for r in res.trace])
        first = min(mism) - 1 if mism else min(len(errs), len(ref_errs))
        assert first >= t + 2, "the hooked step and the two after it must be compared"
        dev = float(np.max(np.abs(errs[:first] - ref_errs[:first])))
        print(f"{name} t={t}: max |relerr - oracle| = {dev:.3e} over {first} iterations, ties {sorted(ties)}")
        assert dev < FIT_ATOL
        if not mism:
            assert len(seq) == len(ref.accepted) and res.stop_reason == ref.stop_reason
            fdev = _rel(res.model.as_vector(), O.stack(ref.factors))
            print(f"  factors rel = {fdev:.3e}")
            assert fdev < FACTOR_RTOL
    # the branch is an overlap, not a different computation: bitwise identical traces and factors
    assert [(r.accepted, r.relerr, r.mu) for r in res0.trace] == [(r.accepted, r.relerr, r.mu) for r in res1.trace]
    assert np.array_equal(res0.model.as_vector(), res1.model.as_vector())
