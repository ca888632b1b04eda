# end-of-round evidence (4-GPU box): GPU suite incl. 2-GPU tests, smoke, headline line + reference arm (GPU 0),
# multi-process parity, N=2/4 lines of every config
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?; grep "^{" gpurun_out/bench_final.log > gpurun_out/bench_final.json
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; grep "^{" gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
python scripts/line_summary.py gpurun_out/bench_final.json 2>/dev/null | head -4
CUDA_VISIBLE_DEVICES=0 bash scripts/r02_cfg.sh c3 1 3
bash scripts/mg_parity.sh 4
CUDA_VISIBLE_DEVICES=0,1 bash scripts/mg_parity.sh 2
for c in c2 c3 c4; do bash scripts/r02_cfg.sh $c 4 3; CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh $c 2 3; done
bash scripts/r02_cfg.sh c5 4 2
