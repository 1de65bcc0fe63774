"""TATN matrix IO (matrix_io.hpp) and the CLI's exit-code contract.

CPU: the writer is byte-identical to the reference's own write_matrix_binary / _csv, the
reference reads our files and we read its files, error cases match; usage errors exit 2;
predict prints the reference's closed forms. GPU: verify on golden directories made by the
oracle exits 0, and exits 1 once an expected vector is perturbed.
"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2205_14135_b200 import cli, iomodel, tatn_io

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden" / "tatn_causal_n256_d64"
need_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref (the reference compiled here) not built")


def _edge_matrix():
    m = np.random.default_rng(3).standard_normal((7, 5)) * np.logspace(-300, 300, 35).reshape(7, 5)
    m[0, 0], m[0, 1], m[0, 2], m[0, 3] = np.inf, -np.inf, -0.0, 5e-324
    return m


@need_ref
@pytest.mark.parametrize("binary", [True, False])
def test_writer_bytes_match_reference(tmp_path, binary):
    m = _edge_matrix()
    ext = "tatn" if binary else "csv"
    O.ref_write_matrix(tmp_path / f"ref.{ext}", m, binary)
    (tatn_io.write_matrix_binary if binary else tatn_io.write_matrix_csv)(m, tmp_path / f"ours.{ext}")
    assert (tmp_path / f"ref.{ext}").read_bytes() == (tmp_path / f"ours.{ext}").read_bytes()


@need_ref
@pytest.mark.parametrize("binary", [True, False])
def test_cross_read(tmp_path, binary):
    m = _edge_matrix()
    ext = "tatn" if binary else "csv"
    (tatn_io.write_matrix_binary if binary else tatn_io.write_matrix_csv)(m, tmp_path / f"ours.{ext}")
    back = O.ref_read_matrix(tmp_path / f"ours.{ext}", binary)
    assert back.tobytes() == m.tobytes()
    O.ref_write_matrix(tmp_path / f"ref.{ext}", m, binary)
    ours = (tatn_io.read_matrix_binary if binary else tatn_io.read_matrix_csv)(tmp_path / f"ref.{ext}")
    assert ours.tobytes() == m.tobytes()


def test_roundtrip_and_errors(tmp_path):
    m = _edge_matrix()
    tatn_io.write_matrix_binary(m, tmp_path / "a.tatn")
    assert tatn_io.read_matrix_binary(tmp_path / "a.tatn").tobytes() == m.tobytes()
    tatn_io.write_matrix_csv(m, tmp_path / "a.csv")
    assert tatn_io.read_matrix_csv(tmp_path / "a.csv").tobytes() == m.tobytes()
    buf = (tmp_path / "a.tatn").read_bytes()
    for bad, what in ((b"TATX" + buf[4:], "magic"), (buf[:10], "header"), (buf[:-1], "payload")):
        (tmp_path / "bad.tatn").write_bytes(bad)
        with pytest.raises(tatn_io.MatrixIOError, match=what):
            tatn_io.read_matrix_binary(tmp_path / "bad.tatn")
    (tmp_path / "r.csv").write_text("1,2\n3\n")
    with pytest.raises(tatn_io.MatrixIOError, match="ragged"):
        tatn_io.read_matrix_csv(tmp_path / "r.csv")
    (tmp_path / "e.csv").write_text("\n\n")
    with pytest.raises(tatn_io.MatrixIOError, match="empty"):
        tatn_io.read_matrix_csv(tmp_path / "e.csv")
    # blanks and CR are trimmed, empty lines skipped (matrix_io.cpp:82-113)
    (tmp_path / "w.csv").write_text(" 1.5 ,\t2\r\n\n3,4\n")
    assert tatn_io.read_matrix_csv(tmp_path / "w.csv").tolist() == [[1.5, 2.0], [3.0, 4.0]]


@need_ref
def test_reference_rejects_what_we_reject(tmp_path):
    (tmp_path / "bad.tatn").write_bytes(b"TATX\x01\x00\x00\x00\x01\x00\x00\x00" + bytes(8))
    with pytest.raises(RuntimeError):
        O.ref_read_matrix(tmp_path / "bad.tatn", True)
    (tmp_path / "r.csv").write_text("1,2\n3\n")
    with pytest.raises(RuntimeError):
        O.ref_read_matrix(tmp_path / "r.csv", False)


def test_golden_fixture_is_well_formed():
    meta = json.loads((GOLDEN / "meta.json").read_text())
    n, d = meta["n"], meta["d"]
    for name in ("q", "k", "v", "do", "o", "dq", "dk", "dv"):
        assert tatn_io.read_matrix_binary(GOLDEN / f"{name}.tatn").shape == (n, d)
    assert tatn_io.read_matrix_binary(GOLDEN / "lse.tatn").shape == (n, 1)
    q = tatn_io.read_matrix_binary(GOLDEN / "q.tatn")
    assert np.array_equal(O.round_to(q, meta["dtype"]), q)  # inputs stored already rounded


@pytest.mark.parametrize("argv", [
    ["verify", "--golden", "x", "--p-drop", "1.0"],
    ["predict", "--n", "0"],
    ["sweep", "--out", "x.csv", "--mask", "diagonal"],
    ["frobnicate"],
    ["verify"],
    ["predict", "--d", "abc"],
])
def test_usage_errors_exit_2(argv):
    assert cli.main(argv) == 2


def test_config_file_and_precedence(tmp_path):
    cfg = tmp_path / "c.cfg"
    cfg.write_text("# comment\nn = 256\nd=64\nm=65536\n")
    assert cli.main(["predict", "--config", str(cfg)]) == 0
    (tmp_path / "bad.cfg").write_text("n=256\nwidth=3\n")
    assert cli.main(["predict", "--config", str(tmp_path / "bad.cfg")]) == 2
    (tmp_path / "p.cfg").write_text("p_drop=1.5\n")
    assert cli.main(["predict", "--config", str(tmp_path / "p.cfg")]) == 2
    assert cli.main(["predict", "--config", str(tmp_path / "p.cfg"), "--p-drop", "0.1"]) == 0  # flag overrides


def test_predict_matches_closed_forms(capsys):
    assert cli.main(["predict", "--n", "1024", "--d", "64", "--m", "65536"]) == 0
    row = capsys.readouterr().out.strip().splitlines()[1].split(",")
    assert row[:5] == ["1024", "64", "65536", "256", "64"]
    assert (int(row[5]), int(row[6])) == (4390912, 2162688)  # SPEC.md:331 (io_predict.hpp:29)
    plan = iomodel.plan_tiles(1024, 64, 65536)
    assert (int(row[7]), int(row[8])) == iomodel.predict_flash_forward_io(1024, 64, plan)


def test_module_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_2205_14135_b200.cli", "predict", "--n", "1", "--d", "1",
                        "--m", "64"], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_verify_committed_golden():
    assert cli.main(["verify", "--golden", str(GOLDEN)]) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,mask,dtype", [(200, 64, "none", "bf16"), (384, 128, "causal", "fp16"),
                                            (256, 64, "padding:197", "bf16")])
def test_verify_generated_golden(tmp_path, n, d, mask, dtype):
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    import make_tatn

    g = make_tatn.make(tmp_path / "g", n, d, mask, dtype)
    assert cli.main(["verify", "--golden", str(g)]) == 0
    # dump -> the GPU outputs as TATN, read back by the reference's reader when available
    assert cli.main(["dump", "--golden", str(g), "--out", str(tmp_path / "gpu")]) == 0
    got = tatn_io.read_matrix_binary(tmp_path / "gpu" / "dk.tatn")
    if O.have_ref():
        assert O.ref_read_matrix(tmp_path / "gpu" / "dk.tatn", True).tobytes() == got.tobytes()
    # a perturbed expectation fails with exit 1
    bad = tmp_path / "bad"
    shutil.copytree(g, bad)
    o = tatn_io.read_matrix_binary(bad / "o.tatn")
    o[3, 5] += 0.5
    tatn_io.write_matrix_binary(o, bad / "o.tatn")
    assert cli.main(["verify", "--golden", str(bad)]) == 1


@pytest.mark.gpu
def test_sweep_csv(tmp_path):
    out = tmp_path / "runs.csv"
    assert cli.main(["sweep", "--n", "256,512", "--d", "64", "--mask", "causal", "--repeats", "2",
                     "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == ",".join(cli.RUN_RECORD)
    assert len(lines) == 3
