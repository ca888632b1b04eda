# configs[2] graph-rebuild check: the graph kernels' parity tests, the c3 line
# at N = 1, and an ncu launch list of the graph-stream kernels of one epoch
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "laplacian or transpose or apply or materializer or stream" \
    > gpurun_out/graph_tests.log 2>&1; echo graph tests rc=$?
tail -2 gpurun_out/graph_tests.log
timeout 1500 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/c3_n1.log 2>&1; echo c3 rc=$?
grep '^{' gpurun_out/c3_n1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],1), '%.4g' % d['value'], 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), d['cpu_baseline'] and d['cpu_baseline']['value'])
for k,v in list(d['kernels'].items())[:10]: print('  ', k, round(v['ms_total']/d['steps'],2), v['launches']//d['steps'])" || tail -5 gpurun_out/c3_n1.log
CMD="python bench.py --config c3 --steps 1 --warmup 1 --skip-e2e --skip-cpu"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"lap_|transpose_|seg_sort|delta_|inv_sqrt|scan_|col_hist|zero_i32" -c 3000 --csv \
    --log-file gpurun_out/c3_graph_launches.csv $CMD > gpurun_out/c3_graph_ncu.log 2>&1; echo ncu rc=$?
