"""Pin the oracle's ALS restatement (oracle/cp_oracle.py: pinv_psd, als_step, als_line_search_step,
fit_als) against fixtures captured from the reference (tests/golden/make_als_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import cp_oracle as O
from tests import _golden as G


def test_golden_recorded_bitwise_oracle():
    assert bool(G.als_units()["oracle_bitwise"])
    for name, c in G.als_fits().items():
        assert bool(c["oracle_bitwise"]), name


@pytest.mark.parametrize("name", sorted(k for k in G.als_units() if k.startswith("pinv_")))
def test_oracle_pinv_psd(name):
    c = G.als_units()[name]
    np.testing.assert_array_equal(O.pinv_psd(c["in"]), c["out"])


@pytest.mark.parametrize("name", sorted(k for k in G.als_units() if k.startswith("step")))
def test_oracle_als_steps(name):
    c = G.als_units()[name]
    dims = tuple(int(x) for x in c["dims"])
    r = int(c["rank"])
    start = G.split_stacked(c["start"], dims, r)
    hist = G.split_stacked(c["hist"], dims, r)
    np.testing.assert_array_equal(O.stack(O.als_step(c["y"], start)), c["als"])
    for t in (1, 2, 5):
        np.testing.assert_array_equal(O.stack(O.als_line_search_step(c["y"], start, hist, t)), c[f"ls_t{t}"])
    np.testing.assert_array_equal(O.stack(O.als_line_search_step(c["y"], start, None, 3)), c["ls_nohist"])


@pytest.mark.parametrize("name", sorted(G.als_fits()))
def test_oracle_fit_als(name):
    from paper_1205_2584_b200 import synth

    c = G.als_fits()[name]
    cfg = G.als_config(name, c)
    y = synth.make_tensor(cfg, 0)
    assert synth.tensor_digest(y) == str(c["digest"])
    variant = name.rsplit("_", 1)[1]
    res = O.fit_als(y, O.OracleConfig(rank=cfg.rank, variant=variant, tol=float(c["tol"]),
                                       max_iters=int(c["max_iters"]), seed=0))
    tr = np.array([[t, e, m, float(a)] for (t, e, m, a) in res.trace])
    np.testing.assert_array_equal(tr, c["trace"])
    assert res.stop_reason == str(c["stop"])
    np.testing.assert_array_equal(O.stack(res.factors), c["factors"])
