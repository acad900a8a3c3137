"""CPTN format, run records and MedSAE (CPU), pinned to files and scores produced by the
reference itself (tests/golden/make_cptn_golden.py).  Mirrors the reference's test_cptn.py cases:
round trips, deterministic bytes, header layout, bad magic / version / kind, truncation,
metadata comments."""

import json
import struct

import numpy as np
import pytest

from paper_1205_2584_b200 import cptn, records
from paper_1205_2584_b200.tensor import DenseTensor, KruskalModel

from tests.conftest import GOLDEN


@pytest.mark.parametrize("name", ["cptn_real.cptn", "cptn_complex.cptn", "cptn_matrix.cptn"])
def test_reads_reference_files_and_rewrites_identical_bytes(tmp_path, name):
    src = GOLDEN / name
    t = cptn.read_tensor(src)
    out = tmp_path / name
    cptn.write_tensor(out, t)
    assert out.read_bytes() == src.read_bytes()


def test_header_parse(tmp_path):
    h = cptn.read_header(GOLDEN / "cptn_complex.cptn")
    assert (h.kind, h.dims, h.payload_offset) == (1, (2, 3, 2), 16 + 3 * 8)
    raw = (GOLDEN / "cptn_real.cptn").read_bytes()
    assert raw[:4] == b"CPTN" and struct.unpack("<I", raw[4:8])[0] == 1 and raw[8] == 0 and raw[9] == 3
    assert raw[10:16] == bytes(6)


def test_roundtrip_real_and_complex_column_major(tmp_path):
    rng = np.random.default_rng(0)
    for arr in (rng.standard_normal((4, 3, 2, 2)), rng.standard_normal((5, 6)) + 1j * rng.standard_normal((5, 6))):
        p = tmp_path / "t.cptn"
        cptn.write_tensor(p, DenseTensor(arr))
        back = cptn.read_tensor(p)
        assert back.dims == arr.shape and np.array_equal(back.data, arr)
        flat = np.frombuffer(p.read_bytes()[16 + 8 * arr.ndim:], dtype="<c16" if np.iscomplexobj(arr) else "<f8")
        assert np.array_equal(flat, arr.reshape(-1, order="F"))


def _corrupt(tmp_path, edit):
    raw = bytearray((GOLDEN / "cptn_real.cptn").read_bytes())
    raw = edit(raw)
    p = tmp_path / "bad.cptn"
    p.write_bytes(bytes(raw))
    return p


def test_format_errors(tmp_path):
    with pytest.raises(cptn.FormatError, match="bad magic"):
        cptn.read_tensor(_corrupt(tmp_path, lambda r: b"XPTN" + r[4:]))
    with pytest.raises(cptn.FormatError, match="unsupported version 2"):
        cptn.read_tensor(_corrupt(tmp_path, lambda r: r[:4] + struct.pack("<I", 2) + r[8:]))
    with pytest.raises(cptn.FormatError, match="unknown scalar kind 7"):
        cptn.read_tensor(_corrupt(tmp_path, lambda r: r[:8] + bytes([7]) + r[9:]))
    with pytest.raises(cptn.FormatError, match="truncated header"):
        cptn.read_tensor(_corrupt(tmp_path, lambda r: r[:10]))
    with pytest.raises(cptn.FormatError, match="truncated dims"):
        cptn.read_tensor(_corrupt(tmp_path, lambda r: r[:20]))
    with pytest.raises(cptn.FormatError, match="expected 60 scalars, found 59"):
        cptn.read_tensor(_corrupt(tmp_path, lambda r: r[:-8]))
    assert issubclass(cptn.FormatError, ValueError)


def test_matrix_helpers_and_metadata(tmp_path):
    m = cptn.read_matrix(GOLDEN / "cptn_matrix.cptn")
    assert m.shape == (4, 2)
    with pytest.raises(cptn.FormatError, match="expected a matrix, got order 3"):
        cptn.read_matrix(GOLDEN / "cptn_real.cptn")
    meta = cptn.read_metadata(GOLDEN / "cptn_meta.meta")
    assert meta == {"dims": "3,4,5", "R": "2", "nu": "0.5", "snr_db": "inf"}
    p = tmp_path / "m.meta"
    cptn.write_metadata(p, {"dims": "3,4,5", "R": 2, "nu": 0.5, "snr_db": "inf"})
    assert p.read_bytes() == (GOLDEN / "cptn_meta.meta").read_bytes()
    p.write_text("# comment\n\n key = value \nx=1=2\n", encoding="utf-8")
    assert cptn.read_metadata(p) == {"key": "value", "x": "1=2"}


def test_record_csv_matches_reference_bytes(tmp_path):
    recs = [records.RunRecord(3, float("nan"), 4, None, "auto", 17, 12, 123.456, 0.0123456789, -45.5, None, "tol"),
            records.RunRecord(0, 0.5, 2, float("inf"), "flm-b", 0, 0, 0.0, float("nan"), None, None, "error")]
    p = tmp_path / "r.csv"
    records.write_csv(p, recs)
    assert p.read_bytes() == (GOLDEN / "record_case.csv").read_bytes()
    with pytest.raises(ValueError):
        records.RunRecord(0, 0.5, 2, None, "auto", 3, 4, 0.0, 0.1, None, None, "tol")


def test_medsae_matches_reference():
    z = np.load(GOLDEN / "medsae_case.npz")
    ref = json.load(open(GOLDEN / "medsae_case.json"))
    truth = KruskalModel([z[f"truth{n}"] for n in range(3)])
    for key in ("perturbed", "exact"):
        est = KruskalModel([z[f"{'est' if key == 'perturbed' else 'exact'}{n}"] for n in range(3)])
        got = records.medsae_pair(truth, est)
        assert got["first_db"] == pytest.approx(ref[key]["first_db"], abs=1e-9)
        assert got["rest_db"] == pytest.approx(ref[key]["rest_db"], abs=1e-9)
    assert ref["exact"]["first_db"] == -300.0
