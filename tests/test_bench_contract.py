"""The bench's JSON-line contract (bench.py docstring), checked on the recorded B200 lines in
profiles/ (CPU only: the lines were produced on the GPU box by scripts/gpu_profile.sh) and on
the CLI surface of bench.py."""
import json
import math
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
LATEST = sorted(ROOT.glob("profiles/r[0-9][0-9]*_bench_ours.json"))[-1]  # latest recorded run


def _line(path):
    lines = [l for l in path.read_text().splitlines() if l.strip()]
    assert len(lines) == 1, f"{path}: exactly one JSON line expected"
    return json.loads(lines[0])


def test_our_line_has_every_contract_key():
    d = _line(LATEST)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
                "cpu_baseline", "clocks"):
        assert key in d, key
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["gpu_launches"] == 4 * d["steps"]  # K1 | K2 K3 K4 per step
    assert "workload" in d["config"]
    e2e = d["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0 and 0 < e2e["value"] < d["value"]
    rl = d["roofline"]
    assert rl["bound"] in ("hbm", "tensor") and rl["unit"] in ("GB/s", "TFLOP/s")
    assert math.isclose(rl["frac"], rl["achieved"] / rl["peak"], rel_tol=1e-3)
    assert 0 < rl["frac"] < 1
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad & set(d["clocks"]["reasons"])


def test_reference_line_matches_our_metric():
    ours = _line(LATEST)
    ref = _line(pathlib.Path(str(LATEST).replace("_bench_ours", "_bench_ref")))
    assert ref["impl"] == "reference"
    for key in ("metric", "unit", "higher_is_better"):
        assert ref[key] == ours[key], key
    assert ref["config"]["workload"] == ours["config"]["workload"]
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["cpu_baseline"]["value"] == ref["value"]


def test_bench_cli_parses_its_flags():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120, cwd=ROOT)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl"):
        assert flag in out.stdout, flag
