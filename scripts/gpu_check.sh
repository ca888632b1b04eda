set -x
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py --steps 2 --warmup 1 --skip-cpu > gpurun_out/bench1.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/pytest_gpu.log
tail -c 3000 gpurun_out/bench1.log
