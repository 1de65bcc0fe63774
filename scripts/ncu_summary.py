"""Summarise ncu reports (gpurun_out/*.ncu-rep) into profiles/<round>_ncu_summary.{json,md}
and merge the per-kernel DRAM traffic into profiles/ncu_summary.json (read by bench.py)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "smsp__inst_executed.sum": "instructions",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_lsu_pct",
}
SCALE = {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "Ghz": 1e9, "Mhz": 1e6}


def read(rep):
    """Metrics of an .ncu-rep, or of its `ncu -i REP --page raw --csv` export (*_raw.csv)."""
    if str(rep).endswith(".csv"):
        out = Path(rep).read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, res = rows[0], rows[1], {}
    name_col = hdr.index("Kernel Name")
    for vals in rows[2:]:
        k = {"kernel": vals[name_col][:80]}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                k[key] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        res.setdefault("launches", []).append(k)
    return res


def main():
    tag = sys.argv[1]
    reps = sys.argv[2:]
    summary = {}
    for r in reps:
        summary[Path(r).stem.replace("_raw", "")] = read(r)
    (ROOT / "profiles" / f"{tag}_ncu_summary.json").write_text(json.dumps(summary, indent=1))
    # merge per-launch DRAM traffic into profiles/ncu_summary.json (bench.py's roofline "traffic")
    merged_f = ROOT / "profiles" / "ncu_summary.json"
    merged = json.loads(merged_f.read_text()) if merged_f.exists() else {"workloads": {}}
    names = {"gpt2": "gpt2-small", "16k": "long-16k", "bert": "bert-large"}
    for rep_name, s in summary.items():
        parts = rep_name.split("_")  # prof_{fwd|bwd}_{gpt2|16k}
        if len(parts) != 3 or parts[1] not in ("fwd", "bwd") or parts[2] not in names or not s.get("launches"):
            continue
        k = s["launches"][0]
        merged["workloads"].setdefault(names[parts[2]], {})["fwd_K1" if parts[1] == "fwd" else "bwd_K3"] = {
            "dram_bytes_per_launch": k.get("dram_read", 0) + k.get("dram_write", 0),
            "duration_ms_ncu": k.get("duration", 0) * 1e3,
            "tensor_pipe_active_pct": k.get("tensor_pipe_active_pct"),
            "source": f"profiles/{tag}_ncu_summary.json ({rep_name}, ncu --set full, 1 launch, cold cache)"}
    merged_f.write_text(json.dumps(merged, indent=1))
    lines = [f"# ncu summary {tag}", "", "| report | kernel | ms | DRAM read GB | DRAM write GB | tensor pipe % | SM thru % | XU % | smem TC % | smem LSU % |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for name, s in summary.items():
        for k in s["launches"]:
            lines.append(f"| {name} | {k['kernel'][:40]} | {k.get('duration', 0) * 1e3:.4f} | "
                         f"{k.get('dram_read', 0) / 1e9:.3f} | {k.get('dram_write', 0) / 1e9:.3f} | "
                         f"{k.get('tensor_pipe_active_pct', 0):.1f} | {k.get('sm_throughput_pct', 0):.1f} | "
                         f"{k.get('xu_pipe_pct', 0):.1f} | {k.get('smem_tc_pct', 0):.1f} | {k.get('smem_lsu_pct', 0):.1f} |")
    (ROOT / "profiles" / f"{tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
