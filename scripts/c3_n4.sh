# configs[2] at N = 4 (gpurun --gpus 4), then the ncu launch list of the graph-stream kernels at N = 1
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 \
    bench.py --config c3 --gpus 4 --steps 3 --warmup 3 --skip-cpu > gpurun_out/c3_n4.log 2>&1; echo n4 rc=$?
grep '^{' gpurun_out/c3_n4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],1), '%.4g' % d['value'], 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1))
for k,v in list(d['kernels'].items())[:8]: print('  ', k, round(v['ms_total']/d['steps'],2), v['launches']//d['steps'])" || tail -5 gpurun_out/c3_n4.log
CMD="python bench.py --config c3 --steps 1 --warmup 1 --skip-e2e --skip-cpu"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"lap_|transpose_|seg_sort|delta_|inv_sqrt|scan_|col_hist|zero_i32|hub_rows|gcn_fwd" -c 3000 --csv \
    --log-file gpurun_out/c3_graph_launches.csv $CMD > gpurun_out/c3_graph_ncu.log 2>&1; echo ncu rc=$?
