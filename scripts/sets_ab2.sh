for k in 4 3; do
  DGNN_BLOCK0_SETS=$k timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/bs_c3$k.log 2>&1
  echo "c3 sets=$k $(grep '^{' gpurun_out/bs_c3$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), d["hbm_peak_gb"])')"
done
DGNN_BLOCK0_SETS=3 timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/c3_tl1.log 2>&1
