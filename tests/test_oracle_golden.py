"""Pin the CPU oracle (oracle/cp_oracle.py) against the golden fixtures captured from the
reference implementation itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import cp_oracle as O
from tests import _golden as G


@pytest.mark.parametrize("cname", sorted(G.unit_cases()))
def test_oracle_building_blocks(cname):
    c = G.unit_cases()[cname]
    dims = tuple(int(x) for x in c["dims"])
    r = int(c["rank"])
    fac = G.split_stacked(c["factors"], dims, r)
    y = np.asfortranarray(c["y"])
    M = np.concatenate([O.mttkrp(y, fac, n).reshape(-1, order="F") for n in range(1, len(dims) + 1)])
    np.testing.assert_allclose(M, c["mttkrp"], rtol=1e-13, atol=1e-13)
    g = O.gram_cache(fac)
    np.testing.assert_allclose(np.concatenate([x.reshape(-1, order="F") for x in g.C]), c["grams"], atol=1e-13)
    assert abs(O.relative_error(y, fac) - float(c["relerr"])) < 1e-13
    np.testing.assert_allclose(O.stack(O.normalize_equal_energy(fac)), c["nee"], atol=1e-13)
    Ms = [O.mttkrp(y, fac, n) for n in range(1, len(dims) + 1)]
    for mu in (1e-4, 0.1, 10.0):
        for variant in ("auto", "flm-a", "flm-b"):
            for refine in (0, 2):
                key = f"step_{variant}_{mu:g}_{refine}"
                if key + "_error" in c:
                    with pytest.raises(np.linalg.LinAlgError):
                        O.flm_candidate(fac, mu, variant, g, Ms, refine)
                    continue
                got = O.stack(O.flm_candidate(fac, mu, variant, g, Ms, refine))
                base = O.stack(fac)
                d_ref = c[key] - base
                assert np.linalg.norm((got - base) - d_ref) <= 1e-10 * max(np.linalg.norm(d_ref), 1e-300)


@pytest.mark.parametrize("name", G.fit_names(include_full=False))
def test_oracle_reproduces_reference_trace(name):
    from paper_1205_2584_b200 import synth

    d = G.load_fit(name)
    y = synth.make_tensor(G.synth_config(d), d["seed"])
    res = O.fit_lm(y, O.OracleConfig(rank=d["rank"], variant=d["variant"], tau=d["tau"], tol=d["tol"],
                                      max_iters=d["max_iters"], seed=d["seed"]))
    tr = np.array([[t, e, m, float(a)] for (t, e, m, a) in res.trace])
    assert tr.shape == d["trace"].shape
    assert G.accept_seq(tr) == G.accept_seq(d["trace"])
    assert res.stop_reason == d["stop_reason"]
    np.testing.assert_allclose(tr[:, 1], d["trace"][:, 1], rtol=0, atol=1e-12)
    np.testing.assert_allclose(tr[:, 2], d["trace"][:, 2], rtol=1e-12)
    v = O.stack(res.factors)
    assert np.linalg.norm(v - d["factors"]) <= 1e-10 * np.linalg.norm(d["factors"])


@pytest.mark.parametrize("key", sorted(G.ensemble())[:8])
def test_oracle_ensemble(key):
    e = G.ensemble()[key]
    variant = key.split("_", 1)[1]
    res = O.fit_lm(e["y"], O.OracleConfig(rank=int(e["rank"]), variant=variant, tol=1e-10, max_iters=40,
                                          seed=int(e["seed"])))
    assert res.stop_reason == str(e["stop"])
    tr = np.array([[t, er, m, float(a)] for (t, er, m, a) in res.trace])
    np.testing.assert_allclose(tr[:, 1], e["trace"][:, 1], atol=1e-12)


def test_nielsen_known_answers():
    # the reference's own known answers (tests/test_solver.py:195-209 in the reference)
    mu, growth, ok = O.nielsen(1.0, 2.0, 1.0)
    assert np.isclose(mu, 1.0 / 3.0) and growth == 2.0 and ok
    assert np.isclose(O.nielsen(1.0, 2.0, 0.5)[0], 1.0)
    mu, growth, ok = O.nielsen(1.0, 2.0, -1.0)
    assert (mu, growth, ok) == (2.0, 4.0, False)
    assert O.nielsen(mu, growth, -1.0)[:2] == (8.0, 8.0)


def test_dense_step_equivalence_small():
    rng = np.random.default_rng(8)
    fac = [rng.standard_normal((d, 2)) for d in (3, 4, 5)]
    for f in fac:
        f /= np.linalg.norm(f, axis=0, keepdims=True)
    y = np.asfortranarray(O.reconstruct(fac) + 0.1 * rng.standard_normal((3, 4, 5)))
    g = O.gram_cache(fac)
    M = [O.mttkrp(y, fac, n) for n in (1, 2, 3)]
    for mu in (1e-4, 0.1, 10.0):
        ref = O.dense_damped_step(y, fac, mu)
        for variant in ("flm-a", "flm-b"):
            d = O.stack(O.flm_candidate(fac, mu, variant, g, M)) - O.stack(fac)
            assert np.linalg.norm(d - ref) / np.linalg.norm(ref) < 1e-8
