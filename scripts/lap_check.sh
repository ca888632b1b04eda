timeout 1500 python -m pytest tests -q -m gpu -x -k "lap or Lap or smooth or graph or c3 or delta or materi or csr" 2>&1 | tail -2
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/lap_c3.log 2>&1; grep '^{' gpurun_out/lap_c3.log > gpurun_out/lap_c3.json; python scripts/line_summary.py gpurun_out/lap_c3.json 2>/dev/null | head -1
