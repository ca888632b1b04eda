# final one-GPU evidence with the final code: GPU suite, smoke, headline line (+CPU baseline, e2e), reference arm,
# configs[2] / [3] lines at N=1 (with e2e)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?; grep "^{" gpurun_out/bench_final.log > gpurun_out/bench_final.json
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; grep "^{" gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
python scripts/line_summary.py gpurun_out/bench_final.json 2>/dev/null | head -4
bash scripts/r02_cfg.sh c3 1 3
bash scripts/r02_cfg.sh c4 1 2
