timeout 1500 python -m pytest tests -q -m gpu -x -k "lap or Lap or smooth or graph or c3 or delta or materi or csr or transpose or apply or golden or residency or epoch or reference or first_layer" 2>&1 | tail -1
for c in c3 c2; do
timeout 900 python bench.py --config $c --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/g2_$c.log 2>&1; grep '^{' gpurun_out/g2_$c.log > gpurun_out/g2_$c.json; python scripts/line_summary.py gpurun_out/g2_$c.json 2>/dev/null | head -1
done
