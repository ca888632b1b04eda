# graph-stream priority A/B on c3 and c2 (N=1)
for c in c3 c2; do for p in -1 0; do
  DGNN_GRAPH_PRIORITY=$p timeout 900 python bench.py --config $c --steps 4 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/pr_$c$p.log 2>&1
  echo "$c prio=$p $(grep '^{' gpurun_out/pr_$c$p.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],1), d["clocks"]["sm_mhz"])')"
done; done
