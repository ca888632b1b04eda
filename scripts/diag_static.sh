# compute-only epoch (graphs of the first epoch kept) vs the measured one, c3 and c2 at N=1
for c in c3 c2; do for d in 0 1; do
  DGNN_DIAG_STATIC_GRAPH=$d timeout 900 python bench.py --config $c --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/ds_$c$d.log 2>&1
  echo "$c static=$d $(grep '^{' gpurun_out/ds_$c$d.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), d["clocks"]["sm_mhz"])')"
done; done
