mkdir -p gpurun_out
python scripts/debug_adam.py > gpurun_out/debug_adam.log 2>&1; echo debug rc=$?
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
