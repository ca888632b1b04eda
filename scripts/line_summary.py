"""Short summary of bench.py JSON lines: python scripts/line_summary.py <file.json> ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f, "unreadable:", exc)
        continue
    e = d.get("e2e") or {}
    r = d.get("roofline") or {}
    print(f, "N", d["n_gpus"], "ms %.1f" % d["ms_per_step"], "value %.4g" % d["value"], "prep %.1f" % d.get("prep_seconds", 0),
          "hbm_peak %.1f GB" % d.get("hbm_peak_gb", 0), "keep", d.get("keep_graphs"), "clocks", d.get("clocks"))
    print("  dominant", r.get("kernel"), r.get("bound"), "frac %.3f" % r.get("frac", 0), "hbm_frac %.3f" % r.get("hbm_frac", 0),
          "3xtf32 %.3f" % r.get("frac_3xtf32_ceiling", 0))
    sp = d.get("spmm_roofline") or {}
    print("  spmm", sp.get("kernel"), "frac", sp.get("frac"), "isolated", (sp.get("isolated") or {}).get("frac"))
    print("  e2e ms", e.get("ms_per_step"), "delta", e.get("delta_vs_full_bytes"), e.get("delta_vs_full_bytes_reference_schedule"),
          "pcie", (e.get("pcie") or {}).get("frac"), "nvlink", d.get("nvlink") and {k: d["nvlink"][k] for k in ("achieved_gbs", "frac", "share_of_step_copying")})
    for k, v in list(d["kernels"].items())[:10]:
        print("   ", k, round(v["ms_total"] / d["steps"], 2), v["launches"] // d["steps"], v.get("hbm_frac") and round(v["hbm_frac"], 3))
