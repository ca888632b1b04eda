"""profiles/<tag>_c3_graph_launches.md from gpurun_out/c3_graph_launches.csv
(scripts/c3_n4.sh: ncu launch list of the graph-stream and aggregation kernels
of `bench.py --config c3 --steps 1 --warmup 1`, serialised, cold-cache).

    python scripts/ncu_c3_graph.py r01
"""

from __future__ import annotations

import collections
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main(tag: str) -> None:
    rows = list(csv.reader(open(ROOT / "gpurun_out" / "c3_graph_launches.csv")))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    t = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0].replace("void ", "").replace("dgnn::", "")
        t[k].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in t.values())
    out = [f"# {tag}: configs[2] graph-stream + aggregation kernels (ncu launch list)", "",
           "`ncu --metrics gpu__time_duration.sum --clock-control none` over the first 3000 matching",
           "launches of `bench.py --config c3 --steps 1 --warmup 1` (prep, warm-up and timed passes;",
           "serialised and cold-cache, so absolute times exceed the bench's).", "",
           f"summed: {tot / 1e6:.1f} ms", "",
           "| kernel | launches | total ms | avg us | max us |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / 1e6:.2f} | {sum(v) / len(v) / 1e3:.1f} | {max(v) / 1e3:.1f} |")
    p = ROOT / "profiles" / f"{tag}_c3_graph_launches.md"
    p.write_text("\n".join(out) + "\n")
    print(p)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
