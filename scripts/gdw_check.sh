timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -m gpu -x -k "gcn or GCN or backward or epoch" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/gdw_c2.log 2>&1; grep '^{' gpurun_out/gdw_c2.log > gpurun_out/gdw_c2.json; python scripts/line_summary.py gpurun_out/gdw_c2.json | head -12
