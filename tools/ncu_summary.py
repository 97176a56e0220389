"""Summarise ncu outputs into committed evidence under profiles/.

    python tools/ncu_summary.py --rep gpurun_out/prof_gains_tc.ncu-rep \
        --launches gpurun_out/launches.csv --tag r01

Writes profiles/<tag>_gains_tc_ncu.md (key metrics of the captured launch),
profiles/<tag>_launches.md (per-kernel time share of the launch list) and
profiles/gains_tc_traffic.json (dram bytes per launch, read by bench.py).
"""

from __future__ import annotations

import argparse
import csv
import io
import re
import json
import subprocess
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tma.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
]


def raw_metrics(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        # section-prefixed names (e.g. "TPC.TriageCompute.sm__...") are
        # keyed by the bare metric name
        m = {}
        for h, v, u in zip(hdr, r, units):
            mm = re.search(r"[a-z0-9]+__.*", h)
            m[mm.group(0) if mm else h] = (v, u)
        res.setdefault(name, m)
    return res


def to_float(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def summarise_rep(rep: Path, tag: str, name_tag: str = "gains_tc"):
    mets = raw_metrics(rep)
    lines = [f"# ncu --set full: {rep.name} ({tag})", ""]
    traffic = None
    for name, m in mets.items():
        lines.append(f"## `{name[:120]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in m:
                lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        rd = m.get("dram__bytes_read.sum")
        wr = m.get("dram__bytes_write.sum")
        if rd and wr and "gains_tc" in name:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                     "Tbyte": 1e12}
            traffic = (to_float(rd[0]) * scale.get(rd[1], 1)
                       + to_float(wr[0]) * scale.get(wr[1], 1))
        lines.append("")
    (ROOT / "profiles" / f"{tag}_{name_tag}_ncu.md").write_text("\n".join(lines))
    if traffic is not None and name_tag == "gains_tc":
        (ROOT / "profiles" / "gains_tc_traffic.json").write_text(json.dumps(
            {"bytes_per_launch": traffic, "source": f"profiles/{tag}_gains_tc_ncu.md",
             "note": "dram__bytes_read.sum + dram__bytes_write.sum of one "
                     "gains_tc_kernel launch (ncu --set full, C4 step)",
             "n": 1000000, "d": 100, "world": 1},
            indent=1) + "\n")
    return traffic


def summarise_launches(path: Path, tag: str):
    text = path.read_text()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0]
        tot[name] += to_float(r[iv])
        cnt[name] += 1
    total = sum(tot.values())
    lines = [f"# ncu launch list ({tag}): gpu__time_duration.sum per kernel",
             "", "cold-cache, serialised by ncu: compare shares, not absolutes",
             "", "| kernel | launches | total ns | share |", "|---|---|---|---|"]
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{name}` | {cnt[name]} | {t:.0f} | {t / total:.4f} |")
    (ROOT / "profiles" / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--name", default="gains_tc")
    a = ap.parse_args()
    if a.rep:
        print("traffic bytes/launch:", summarise_rep(Path(a.rep), a.tag, a.name))
    if a.launches:
        summarise_launches(Path(a.launches), a.tag)


if __name__ == "__main__":
    main()
