# weight-gradient kernels: parity (both variants) + timing at c2 shapes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "weight_grad_tc_long" > gpurun_out/dwts_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/dwts_pytest.log
timeout 600 python scripts/lstm_probe.py --kx 128,68 --steps 8 > gpurun_out/dwts_probe.log 2>&1; echo probe rc=$?
grep -i " dw" gpurun_out/dwts_probe.log
