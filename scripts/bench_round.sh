# full bench line (N=1), the reference arm, and the ncu launch list of the same command
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_full.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-300
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 2500 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
