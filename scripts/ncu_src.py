"""Top stall sites of one ncu capture: python scripts/ncu_src.py rep.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:]]
base = int(data[0]["Address"], 16)
f = lambda d, k: float(d.get(k) or 0)
tot = sum(f(d, "Warp Stall Sampling (All Samples)") for d in data)
print("samples", tot, "warp insts", sum(f(d, "Instructions Executed") for d in data))
for d in sorted(data, key=lambda d: -f(d, "Warp Stall Sampling (All Samples)"))[:n]:
    print(f'{int(d["Address"],16)-base:6x} {f(d,"Warp Stall Sampling (All Samples)")/tot*100:5.1f}% {d["Source"][:80]:80s} {d["Instructions Executed"]}')
