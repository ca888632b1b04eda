# ncu --set full of one launch of kernel $1 inside the bench epoch
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-6} -c 1 -o gpurun_out/full_$1 $CMD > gpurun_out/ncu_$1.log 2>&1; echo full rc=$?
