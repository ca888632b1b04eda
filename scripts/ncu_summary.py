"""Summarise the ncu captures of scripts/profile.sh into profiles/<tag>_*.md.

    python scripts/ncu_summary.py r01
    python scripts/ncu_summary.py r02 c2     # launches_c2.csv, full_c2_*.ncu-rep (scripts/profile_r02.sh)

Reads gpurun_out/launches.csv (per-launch gpu__time_duration + DRAM bytes of
one whole timed epoch, serialised and cold-cache under ncu) and the
gpurun_out/full_<kernel>.ncu-rep captures (`--set full`), writes a launch
table and one page of key metrics per kernel.
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"


def short(name: str) -> str:
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("dgnn::", "")
    return n


def launches(tag: str, src: str = "launches.csv") -> str:
    rows = list(csv.reader(open(OUT / src)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    iK, iM, iV, iU = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    iid = h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        v = float(r[iV].replace(",", ""))
        unit = r[iU]
        if unit in ("usecond",):
            v *= 1e3
        elif unit in ("msecond",):
            v *= 1e6
        elif unit == "Kbyte":
            v *= 1e3
        elif unit == "Mbyte":
            v *= 1e6
        elif unit == "Gbyte":
            v *= 1e9
        per[r[iid]]["name"] = short(r[iK])
        per[r[iid]][r[iM]] = v
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    import json
    (ROOT / "profiles" / f"{tag}_traffic.json").write_text(json.dumps(
        {name: {"launches": n, "avg_us": t / n / 1e3, "dram_bytes_per_launch": b / n}
         for name, (n, t, b) in agg.items()}, indent=1, sort_keys=True) + "\n")
    lines = [f"# {tag}: launch list of one timed epoch (scripts/profile_r02.sh / profile.sh)", "",
             "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none` over exactly the launches of the timed epoch. ncu serialises "
             "launches and starts each cold, so absolute times exceed the bench's; the *share* "
             "column is what the bench's kernel table must agree with.", "",
             f"launches: {len(per)}, summed kernel time: {total / 1e6:.1f} ms", "",
             "| kernel | launches | total ms | share | avg us | DRAM GB/launch | DRAM GB/s |",
             "|---|---:|---:|---:|---:|---:|---:|"]
    for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if t / total < 0.002:
            continue
        lines.append(f"| `{name}` | {n} | {t / 1e6:.2f} | {100 * t / total:.1f}% | {t / n / 1e3:.1f} | "
                     f"{b / n / 1e9:.3f} | {b / t:.0f} |")
    return "\n".join(lines) + "\n"


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "SM Frequency", "Registers Per Thread", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Issue Slots Busy", "Executed Ipc Active",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction"]


def raw_metric(rep: Path, names):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return {}
    h, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for n in names:
        if n in h:
            i = h.index(n)
            out[n] = (vals[i], units[i])
    return out


def kernel_page(tag: str, rep: Path) -> str:
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    iK, iS, iN, iU, iV = (h.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                                "Metric Value"))
    kname = rows[1][iK]
    got = {}
    for r in rows[1:]:
        if r[iN] in WANT and r[iN] not in got:
            got[r[iN]] = f"{r[iV]} {r[iU]}".strip()
    raw = raw_metric(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum",
                           "sm__pipe_tensor_op_utilization.avg.pct_of_peak_sustained_active",
                           "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
                           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                           "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
                           "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
                           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"])
    lines = [f"# {tag}: `{short(kname)}` (`ncu --set full --clock-control none`, one launch of the bench epoch)",
             "", f"full name: `{kname[:200]}`", "", "| metric | value |", "|---|---|"]
    for k in WANT:
        if k in got:
            lines.append(f"| {k} | {got[k]} |")
    for k, (v, u) in raw.items():
        lines.append(f"| `{k}` | {v} {u} |")
    return "\n".join(lines) + "\n"


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    cfg = sys.argv[2] if len(sys.argv) > 2 else None
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    pre = f"full_{cfg}_" if cfg else "full_"
    (prof / f"{tag}_launches.md").write_text(launches(tag, f"launches_{cfg}.csv" if cfg else "launches.csv"))
    for rep in sorted(OUT.glob(pre + "*.ncu-rep")):
        k = rep.stem[len(pre):]
        (prof / f"{tag}_{k}.md").write_text(kernel_page(tag, rep))
    print("\n".join(str(p) for p in sorted(prof.glob(f"{tag}_*"))))


if __name__ == "__main__":
    main()
