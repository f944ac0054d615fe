"""Summarise ncu captures from gpurun_out/ into profiles/ (tracked).

    python scripts/ncu_summarize.py ROUND_TAG [CONFIG]

Reads gpurun_out/launches.csv (the `--metrics gpu__time_duration.sum` launch list) and every
gpurun_out/*_full.ncu-rep (`ncu --set full` captures), and writes per round:
  profiles/<tag>_launches.csv            the launch list (per-kernel durations)
  profiles/<tag>_launch_summary.json     mean duration per kernel and its share of the step
  profiles/<tag>_<name>_ncu.txt          the details page of each full capture
  profiles/<tag>_<name>_ncu.json         key raw metrics (time, dram bytes, pipe utilisation)
and refreshes profiles/attention_ncu_summary_<CONFIG>.json (read by bench.py for roofline.traffic).
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime", "sm__inst_executed_pipe_tensor_subpipe_dmma",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct",
        "sm__inst_executed_pipe_xu", "sm__inst_executed_pipe_fma.avg.pct",
        "sm__inst_executed_pipe_alu.avg.pct", "sm__inst_executed_pipe_fp64.avg.pct",
        "smsp__average_warp_latency_issue_stalled", "smsp__cycles_active.avg")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "s": 1}


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw_metrics(rep: Path) -> dict:
    rows = list(csv.reader(io.StringIO(ncu("-i", str(rep), "--page", "raw", "--csv"))))
    if len(rows) < 3:
        return {}
    hdr, unit, val = rows[0], rows[1], rows[2]
    out = {"kernel": val[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
    for h, u, v in zip(hdr, unit, val):
        if any(h.startswith(k) or k in h for k in KEYS):
            try:
                out[h] = {"unit": u, "value": float(v.replace(",", ""))}
            except ValueError:
                pass
    return out


def to_base(m: dict, name: str):
    e = m.get(name)
    if e is None:
        return None
    return e["value"] * SCALE.get(e["unit"], 1)


def main(tag: str) -> None:
    PROF.mkdir(exist_ok=True)
    launches = OUT / "launches.csv"
    if launches.exists():
        text = launches.read_text()
        body = text[text.index('"ID"'):] if '"ID"' in text else text
        (PROF / f"{tag}_launches.csv").write_text(body)
        rows = list(csv.reader(io.StringIO(body)))
        hdr = rows[0]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        mi = hdr.index("Metric Name")
        agg = collections.OrderedDict()
        byt = collections.defaultdict(float)
        for r in rows[1:]:
            name = r[ki].split("(")[0].replace("void ", "")
            val = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9)
            if r[mi] == "gpu__time_duration.sum":
                agg.setdefault(name, []).append(val)
            elif r[mi].startswith("dram__bytes"):
                byt[name] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        total = sum(sum(v) for v in agg.values())
        summ = {k: {"launches": len(v), "mean_ms": 1e3 * sum(v) / len(v),
                    "share_of_listed": sum(v) / total,
                    "dram_gb_per_launch": byt[k] / len(v) / 1e9 if byt else None}
                for k, v in agg.items()}
        (PROF / f"{tag}_launch_summary.json").write_text(json.dumps(summ, indent=1) + "\n")
        print(json.dumps(summ, indent=1))
    for rep in sorted(OUT.glob("*_full.ncu-rep")):
        name = rep.stem.replace("_full", "")
        (PROF / f"{tag}_{name}_ncu.txt").write_text(ncu("-i", str(rep), "--page", "details"))
        m = raw_metrics(rep)
        t = to_base(m, "gpu__time_duration.sum")
        rd, wr = to_base(m, "dram__bytes_read.sum"), to_base(m, "dram__bytes_write.sum")
        m["summary"] = {"duration_ms": t * 1e3 if t else None,
                        "dram_bytes_per_launch": (rd or 0) + (wr or 0),
                        "dram_gbs": ((rd or 0) + (wr or 0)) / t / 1e9 if t else None}
        (PROF / f"{tag}_{name}_ncu.json").write_text(json.dumps(m, indent=1) + "\n")
        print(name, m["summary"])
        if name.startswith("psa_attn") or name == "attn":
            cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
            (PROF / f"attention_ncu_summary_{cfg}.json").write_text(json.dumps(
                {"source": f"profiles/{tag}_{name}_ncu.json", "kernel": m.get("kernel"),
                 **m["summary"]}, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
