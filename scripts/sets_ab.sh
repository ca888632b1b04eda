# block-0 slot sets 3 vs 2 (keep_graphs), c3 / c2 at N=1; engine tests with 3 sets
timeout 900 python -m pytest tests/test_gpu_engine.py -q -m gpu -x 2>&1 | tail -1
for c in c3 c2; do for k in 3 2; do
  DGNN_BLOCK0_SETS=$k timeout 900 python bench.py --config $c --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/bs_$c$k.log 2>&1
  echo "$c sets=$k $(grep '^{' gpurun_out/bs_$c$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), d["clocks"]["sm_mhz"], d["hbm_peak_gb"])')"
done; done
