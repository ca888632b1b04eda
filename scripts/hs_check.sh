timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -q -m gpu -x 2>&1 | tail -2
for c in c2 c3; do
timeout 900 python bench.py --config $c --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/hs_$c.log 2>&1; grep '^{' gpurun_out/hs_$c.log > gpurun_out/hs_$c.json; python scripts/line_summary.py gpurun_out/hs_$c.json 2>/dev/null | head -1
done
