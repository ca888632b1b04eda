timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -m gpu -x -k "gcn or GCN or epoch or backward or forward" 2>&1 | tail -1
timeout 300 python scripts/gcn_fwd_probe.py
for c in c3 c2; do
timeout 900 python bench.py --config $c --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/k3_$c.log 2>&1; grep '^{' gpurun_out/k3_$c.log > gpurun_out/k3_$c.json; python scripts/line_summary.py gpurun_out/k3_$c.json 2>/dev/null | head -9
done
