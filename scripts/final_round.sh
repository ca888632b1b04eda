# end-of-round check on a 4-GPU box: GPU suite, smoke, bench + reference arm (N = 1),
# configs[2] at N = 4, and the graph-kernel launch list of one c3 epoch (N = 1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_full.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
bash scripts/c3_n4.sh
