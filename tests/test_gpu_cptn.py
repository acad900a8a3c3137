"""GPU: CPTN tensor files streamed straight into device memory (cpf_engine_load_cptn) and the
``fit`` CLI (cpfast/cli.py:95-134 contract) on the engine.  A file-fed fit must equal the
array-fed fit bit for bit (same engine, same bytes on the device), and both match the
reference's golden trace."""

import csv

import numpy as np
import pytest
from click.testing import CliRunner

from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(engine_lib):
    import paper_1205_2584_b200 as api

    return api


def _golden_input(name):
    from paper_1205_2584_b200 import synth

    d = G.load_fit(name)
    cfg = G.synth_config(d)
    return d, synth.make_tensor(cfg, d["seed"])


@pytest.mark.parametrize("name", ["fit_c0_s0_auto", "fit_c3_mini_s0_auto", "fit_c4_mini_s0_auto"])
def test_file_fit_equals_array_fit(api, tmp_path, name):
    from paper_1205_2584_b200 import cptn

    d, y = _golden_input(name)
    path = tmp_path / "y.cptn"
    cptn.write_tensor(path, api.DenseTensor(y))
    conf = api.FitConfig(rank=d["rank"], variant=d["variant"], tau=d["tau"], tol=d["tol"],
                         max_iters=d["max_iters"], seed=d["seed"], init="random")
    a = (api.fit_complex if d["complex_"] else api.fit)(y, conf)
    b = api.fit_file(path, conf, complex_only=bool(d["complex_"]))
    assert [(r.iter, r.relerr, r.mu, r.accepted) for r in a.trace] == [(r.iter, r.relerr, r.mu, r.accepted) for r in b.trace]
    assert np.array_equal(a.model.as_vector(), b.model.as_vector())
    assert b.stop_reason == d["stop_reason"]
    assert abs(b.final_relerr - d["trace"][-1, 1]) < 1e-10


def test_truncated_payload_is_a_format_error(api, tmp_path):
    from paper_1205_2584_b200 import cptn

    _, y = _golden_input("fit_c0_s0_auto")
    path = tmp_path / "y.cptn"
    cptn.write_tensor(path, api.DenseTensor(y))
    raw = path.read_bytes()
    path.write_bytes(raw[:-16])
    with pytest.raises(cptn.FormatError, match=f"expected {y.size} scalars, found {y.size - 2}"):
        api.fit_file(path, api.FitConfig(rank=5, init="random", max_iters=3))


def test_cli_fit_writes_factors_and_record(api, tmp_path):
    from paper_1205_2584_b200 import cptn
    from paper_1205_2584_b200.cli import main
    from paper_1205_2584_b200.records import CSV_COLUMNS

    d, y = _golden_input("fit_c0_s0_auto")
    truth = api.KruskalModel([np.linalg.qr(np.random.default_rng(n).standard_normal((20, 5)))[0] for n in range(3)])
    cptn.write_tensor(tmp_path / "t.cptn", api.DenseTensor(y))
    paths = []
    for n, f in enumerate(truth.factors, start=1):
        cptn.write_matrix(tmp_path / f"t_factor{n}.cptn", f)
        paths.append(str(tmp_path / f"t_factor{n}.cptn"))
    cptn.write_metadata(tmp_path / "t.meta", {"factors": ";".join(paths)})
    res = CliRunner().invoke(main, ["fit", str(tmp_path / "t.cptn"), "--rank", "5", "--init", "random",
                                    "--tau", repr(float(d["tau"])), "--tol", repr(float(d["tol"])),
                                    "--max-iters", str(int(d["max_iters"])), "--truth", str(tmp_path / "t.meta"),
                                    "--out", str(tmp_path / "fitted")], catch_exceptions=False)
    assert res.exit_code == 0, res.output
    assert f"iters={len(d['trace'])} " in res.output and f"stop={d['stop_reason']}" in res.output
    rows = list(csv.reader(open(tmp_path / "fitted.csv")))
    assert rows[0] == list(CSV_COLUMNS)
    rec = dict(zip(rows[0], rows[1]))
    assert abs(float(rec["final_relerr"]) - d["trace"][-1, 1]) < 1e-10
    assert rec["medsae_first_db"] != "" and rec["medsae_rest_db"] != ""
    f1 = cptn.read_matrix(tmp_path / "fitted_factor1.cptn")
    assert f1.shape == (20, 5)


def test_cli_rejects_cpu_only_variants(api, tmp_path):
    """dgn-oracle (the dense desk-scale oracle) stays CPU-only; ALS runs on the engine."""
    from paper_1205_2584_b200 import cptn
    from paper_1205_2584_b200.cli import main

    cptn.write_tensor(tmp_path / "t.cptn", api.DenseTensor(np.ones((3, 3, 3))))
    res = CliRunner().invoke(main, ["fit", str(tmp_path / "t.cptn"), "--rank", "2", "--algo", "dgn-oracle"])
    assert res.exit_code == 1
    assert "not supported on the B200 backend" in res.output


def test_cli_fit_als(api, tmp_path):
    from paper_1205_2584_b200 import cptn
    from paper_1205_2584_b200.cli import main

    rng = np.random.default_rng(3)
    y = np.einsum("ir,jr,kr->ijk", *(rng.standard_normal((d, 2)) for d in (4, 5, 6)))
    cptn.write_tensor(tmp_path / "t.cptn", api.DenseTensor(np.asfortranarray(y)))
    res = CliRunner().invoke(main, ["fit", str(tmp_path / "t.cptn"), "--rank", "2", "--algo", "als-ls",
                                    "--max-iters", "30", "--init", "random"])
    assert res.exit_code == 0, res.output
