"""Command-line harness over the B200 path: golden-vector verification, IO prediction and
sweeps (the reference's bench_cli contract).

    python -m paper_2205_14135_b200.cli verify  --golden DIR [--tol-abs 2e-2 --tol-rel 1e-2]
    python -m paper_2205_14135_b200.cli dump    --golden DIR --out DIR2
    python -m paper_2205_14135_b200.cli predict --n 1024 --d 64 --m 65536
    python -m paper_2205_14135_b200.cli sweep   --n 1024,2048 --d 64 --mask causal --out runs.csv

Exit codes as the reference's: 0 pass, 1 assertion failure, 2 usage error.
Common flags follow SPEC.md:473 (--n --d --m --bc --br --tau --mask {none|causal|padding:<len>}
--p-drop --seed --repeats --out --config <file>); a config file holds `key=value` lines,
flags override it and unknown keys are usage errors.

A golden directory exchanges one head's vectors in the reference's TATN binary format
(matrix_io.hpp:15-16, see tatn_io.py): inputs q, k, v, do (n x d; already rounded to the
16-bit dtype) and expected outputs o, lse (n x 1), dq, dk, dv, plus meta.json
{"n", "nk", "d", "tau", "mask", "dtype", "p_drop", "seed"} and optionally grid (tr x tc 0/1
block mask at 128 x 128). verify runs the sm_100a kernels on the inputs and compares; the
expected vectors come from the CPU oracle (tests/golden/make_tatn.py), never from here.
"""
from __future__ import annotations

import argparse
import csv
import json
import math
import statistics
import sys
from pathlib import Path

import numpy as np

from . import iomodel
from . import tatn_io

EXIT_PASS, EXIT_FAIL, EXIT_USAGE = 0, 1, 2
CONFIG_KEYS = {"n", "d", "m", "bc", "br", "tau", "mask", "p_drop", "seed", "repeats", "out", "golden", "dtype",
               "tol_abs", "tol_rel", "sparsity", "pattern"}
RUN_RECORD = ["algo", "n", "d", "m", "bc", "br", "sparsity", "hbm_read_elems", "hbm_write_elems", "hbm_bytes", "flops",
              "peak_sram_elems", "wall_ms_median", "max_abs_err_vs_oracle"]  # SPEC.md:474, exact order


class UsageError(Exception):
    pass


def _ints(s: str):
    try:
        v = [int(x) for x in str(s).split(",") if x != ""]
    except ValueError as e:
        raise UsageError(f"expected integers, got '{s}'") from e
    if not v:
        raise UsageError("empty list")
    return v


def parse_mask(s: str):
    """--mask {none|causal|padding:<len>} -> (kind, valid_len)."""
    if s in ("none", "causal"):
        return s, None
    if s.startswith("padding:"):
        try:
            ln = int(s.split(":", 1)[1])
        except ValueError as e:
            raise UsageError(f"bad padding length in --mask {s}") from e
        if ln < 0:
            raise UsageError("--mask padding:<len> needs len >= 0")
        return "key_padding", ln
    raise UsageError(f"--mask must be none|causal|padding:<len>, got '{s}'")


def _read_config(path: str) -> dict:
    out = {}
    try:
        lines = Path(path).read_text().splitlines()
    except OSError as e:
        raise UsageError(f"cannot read --config {path}") from e
    for ln in lines:
        ln = ln.strip()
        if not ln or ln.startswith("#"):
            continue
        if "=" not in ln:
            raise UsageError(f"config line without '=': {ln}")
        k, v = (x.strip() for x in ln.split("=", 1))
        k = k.replace("-", "_")
        if k not in CONFIG_KEYS:
            raise UsageError(f"unknown config key '{k}'")
        out[k] = v
    return out


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2205_14135_b200.cli", add_help=True)
    ap.add_argument("command", choices=["verify", "dump", "predict", "sweep"])
    ap.add_argument("--config")
    ap.add_argument("--golden")
    ap.add_argument("--out")
    ap.add_argument("--n")
    ap.add_argument("--d")
    ap.add_argument("--m")
    ap.add_argument("--bc")
    ap.add_argument("--br")
    ap.add_argument("--tau")
    ap.add_argument("--mask")
    ap.add_argument("--p-drop", dest="p_drop")
    ap.add_argument("--seed")
    ap.add_argument("--repeats")
    ap.add_argument("--dtype")
    ap.add_argument("--tol-abs", dest="tol_abs")
    ap.add_argument("--tol-rel", dest="tol_rel")
    ap.add_argument("--sparsity")
    ap.add_argument("--pattern")
    return ap


class _Exit(Exception):
    def __init__(self, code):
        self.code = code


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse exits 2 on its own; keep the code, drop the SystemExit
        sys.stderr.write(f"usage error: {message}\n")
        raise _Exit(EXIT_USAGE)


def resolve(argv):
    ap = build_parser()
    ap.__class__ = _Parser
    ns = ap.parse_args(argv)
    opts = _read_config(ns.config) if ns.config else {}
    for k, v in vars(ns).items():  # flags override the config file
        if k not in ("command", "config") and v is not None:
            opts[k] = v
    return ns.command, opts


def _common(opts):
    p_drop = float(opts.get("p_drop", 0.0))
    if not (0.0 <= p_drop < 1.0):
        raise UsageError(f"--p-drop {p_drop} outside the valid range [0,1)")
    tau = opts.get("tau")
    if tau is not None:
        tau = float(tau)
        if not (tau > 0 and math.isfinite(tau)):
            raise UsageError("--tau must be positive and finite")
    return p_drop, tau


# ----------------------------------------------------------------------------- predict
def cmd_predict(opts) -> int:
    ns, ds = _ints(opts.get("n", "1024")), _ints(opts.get("d", "64"))
    ms = _ints(opts.get("m", "65536"))
    for n in ns:
        for d in ds:
            if n < 1 or d < 1:
                raise UsageError("--n and --d must be >= 1")
    ok = True
    print("n,d,m,bc,br,std_fwd_R,std_fwd_W,flash_fwd_R,flash_fwd_W,std_bwd_R,std_bwd_W,flash_bwd_R,flash_bwd_W,"
          "fwd_ratio,b200_theorem2_bytes_bf16,b200_compulsory_bytes_bf16")
    for n in ns:
        for d in ds:
            for m in ms:
                try:
                    plan = iomodel.plan_tiles(n, d, m, int(opts.get("br", 0) or 0), int(opts.get("bc", 0) or 0))
                except ValueError as e:
                    raise UsageError(str(e)) from e
                sr, sw = iomodel.predict_standard_forward_io(n, d)
                fr, fw = iomodel.predict_flash_forward_io(n, d, plan)
                br_, bw_ = iomodel.predict_standard_backward_io(n, d)
                gr, gw = iomodel.predict_flash_backward_io(n, d, plan)
                t2 = iomodel.theorem2_bound_bytes(n, d, 2, 1, False) + iomodel.theorem2_bound_bytes(n, d, 2, 1, True)
                comp = iomodel.compulsory_bytes(n, d, 2, 1, False) + iomodel.compulsory_bytes(n, d, 2, 1, True)
                ratio = (sr + sw) / max(fr + fw, 1)
                print(f"{n},{d},{m},{plan.bc},{plan.br},{sr},{sw},{fr},{fw},{br_},{bw_},{gr},{gw},{ratio:.4f},{t2},{comp}")
                ok &= all(isinstance(x, int) and x >= 0 for x in (sr, sw, fr, fw, br_, bw_, gr, gw))
    return EXIT_PASS if ok else EXIT_FAIL


# ----------------------------------------------------------------------------- golden runs
def _load_golden(root: Path):
    if not root.is_dir():
        raise UsageError(f"--golden {root} is not a directory")
    try:
        meta = json.loads((root / "meta.json").read_text())
    except (OSError, ValueError) as e:
        raise UsageError(f"{root}/meta.json missing or invalid") from e
    rd = lambda name: tatn_io.read_matrix_binary(root / f"{name}.tatn")
    ins = {k: rd(k) for k in ("q", "k", "v", "do")}
    grid = rd("grid").astype(np.uint8) if (root / "grid.tatn").exists() else None
    return meta, ins, grid


def _run_gpu(meta, ins, grid):
    import torch

    from . import attention as A

    if not torch.cuda.is_available():
        raise RuntimeError("verify needs a CUDA (sm_100) device")
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16}[meta.get("dtype", "bf16")]
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.float32)[None, None].to(dt).cuda()
    q, k, v, do = (dev(ins[x]) for x in ("q", "k", "v", "do"))
    kind, vl = parse_mask(meta.get("mask", "none"))
    spec = A.AttnSpec(mask=kind, tau=meta.get("tau"), p_drop=float(meta.get("p_drop", 0.0)),
                      seed=int(meta.get("seed", 0)))
    if vl is not None:
        spec.valid_len = torch.tensor([vl], dtype=torch.int32, device="cuda")
    if grid is not None:
        spec.block_grid = torch.from_numpy(grid).cuda()
    o, lse = A.flash_fwd(q, k, v, spec)
    dq, dk, dv = A.flash_bwd(q, k, v, o, do, lse, spec)
    torch.cuda.synchronize()
    host = lambda t: t.double().cpu().numpy()[0, 0]
    return {"o": host(o), "lse": host(lse).reshape(-1, 1), "dq": host(dq), "dk": host(dk), "dv": host(dv)}


def _errors(got: np.ndarray, ref: np.ndarray):
    fin = np.isfinite(ref)
    if not np.array_equal(fin, np.isfinite(got)) or not np.array_equal(ref[~fin], got[~fin]):
        return math.inf, math.inf
    g, r = got[fin], ref[fin]
    if g.size == 0:
        return 0.0, 0.0
    mx = float(np.abs(g - r).max())
    den = float(np.linalg.norm(r))
    rel = float(np.linalg.norm(g - r)) / den if den > 0 else (0.0 if mx == 0 else math.inf)
    return mx, rel


def cmd_verify(opts) -> int:
    if "golden" not in opts:
        raise UsageError("verify needs --golden DIR")
    tol_abs, tol_rel = float(opts.get("tol_abs", 2e-2)), float(opts.get("tol_rel", 1e-2))
    root = Path(opts["golden"])
    meta, ins, grid = _load_golden(root)
    _common(meta)
    try:
        got = _run_gpu(meta, ins, grid)
    except RuntimeError as e:
        print(f"verify: {e}")
        return EXIT_FAIL
    ok = True
    for name in ("o", "lse", "dq", "dk", "dv"):
        f = root / f"{name}.tatn"
        if not f.exists():
            continue
        ref = tatn_io.read_matrix_binary(f)
        if ref.shape != got[name].shape:
            print(f"{name}: shape {got[name].shape} != expected {ref.shape}")
            ok = False
            continue
        mx, rel = _errors(got[name], ref)
        good = mx <= tol_abs and rel <= tol_rel
        ok &= good
        print(f"{name}: max_abs={mx:.3e} rel_l2={rel:.3e} {'ok' if good else 'FAIL'}")
    print("verify:", "PASS" if ok else "FAIL", f"(tolerance max_abs <= {tol_abs}, rel_l2 <= {tol_rel})")
    return EXIT_PASS if ok else EXIT_FAIL


def cmd_dump(opts) -> int:
    if "golden" not in opts or "out" not in opts:
        raise UsageError("dump needs --golden DIR --out DIR")
    meta, ins, grid = _load_golden(Path(opts["golden"]))
    got = _run_gpu(meta, ins, grid)
    out = Path(opts["out"])
    out.mkdir(parents=True, exist_ok=True)
    for name, a in got.items():
        tatn_io.write_matrix_binary(a, out / f"{name}.tatn")
    (out / "meta.json").write_text(json.dumps(meta))
    print(f"dump: wrote {', '.join(got)} to {out}")
    return EXIT_PASS


# ----------------------------------------------------------------------------- sweep
def cmd_sweep(opts) -> int:
    import torch

    from . import attention as A

    if "out" not in opts:
        raise UsageError("sweep needs --out <csv>")
    p_drop, tau = _common(opts)
    ns, ds = _ints(opts.get("n", "1024")), _ints(opts.get("d", "64"))
    m = int(opts.get("m", str(iomodel.SMEM_BYTES_PER_CTA // 2)))
    reps = int(opts.get("repeats", "5"))
    if reps < 1:
        raise UsageError("--repeats must be >= 1")
    kind, vl = parse_mask(opts.get("mask", "none"))
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16}[opts.get("dtype", "bf16")]
    if not torch.cuda.is_available():
        print("sweep: needs a CUDA (sm_100) device")
        return EXIT_FAIL
    rows = []
    for n in ns:
        for d in ds:
            if n < 1 or d not in (64, 128):
                raise UsageError("sweep: --n >= 1 and --d in {64, 128} on the B200 path")
            g = torch.Generator(device="cuda").manual_seed(int(opts.get("seed", 0)))
            q, k, v, do = (torch.randn((1, 1, n, d), generator=g, device="cuda").to(dt) for _ in range(4))
            spec = A.AttnSpec(mask=kind, tau=tau, p_drop=p_drop, seed=int(opts.get("seed", 0)))
            if vl is not None:
                spec.valid_len = torch.tensor([min(vl, n)], dtype=torch.int32, device="cuda")
            o, lse = A.flash_fwd(q, k, v, spec)
            A.flash_bwd(q, k, v, o, do, lse, spec)
            times = []
            for _ in range(reps + 1):  # one warm-up discarded
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                o, lse = A.flash_fwd(q, k, v, spec)
                A.flash_bwd(q, k, v, o, do, lse, spec)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            plan = iomodel.plan_tiles(n, d, m)
            fr, fw = iomodel.predict_flash_forward_io(n, d, plan)
            gr, gw = iomodel.predict_flash_backward_io(n, d, plan)
            fl = iomodel.flop_model("flash_forward", n, d, plan) + iomodel.flop_model("flash_backward", n, d, plan)
            rows.append({"algo": "flash_b200", "n": n, "d": d, "m": m, "bc": plan.bc, "br": plan.br,
                         "sparsity": 1.0, "hbm_read_elems": fr + gr, "hbm_write_elems": fw + gw,
                         "hbm_bytes": (fr + gr + fw + gw) * 2, "flops": fl, "peak_sram_elems": plan.working_set,
                         "wall_ms_median": f"{statistics.median(times[1:]):.6f}", "max_abs_err_vs_oracle": ""})
    with open(opts["out"], "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=RUN_RECORD, lineterminator="\n")
        w.writeheader()
        w.writerows(rows)
    print(f"sweep: {len(rows)} rows -> {opts['out']}")
    return EXIT_PASS


def main(argv=None) -> int:
    try:
        cmd, opts = resolve(sys.argv[1:] if argv is None else argv)
        for key in ("n", "d"):
            if key in opts:
                if any(x < 1 for x in _ints(opts[key])):
                    raise UsageError(f"--{key} must be >= 1")
        _common(opts)
        return {"verify": cmd_verify, "dump": cmd_dump, "predict": cmd_predict, "sweep": cmd_sweep}[cmd](opts)
    except _Exit as e:
        return e.code
    except UsageError as e:
        sys.stderr.write(f"usage error: {e}\n")
        return EXIT_USAGE
    except tatn_io.MatrixIOError as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_FAIL


if __name__ == "__main__":
    sys.exit(main())
