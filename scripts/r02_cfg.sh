# one config line at N GPUs: bash scripts/r02_cfg.sh <config> <N> [steps]
C=$1; N=${2:-1}; S=${3:-2}
mkdir -p gpurun_out
if [ "$N" = "1" ]; then
  timeout 2400 python bench.py --config $C --steps $S --warmup 3 --skip-cpu > gpurun_out/r02_${C}_n$N.log 2>&1; echo $C N=$N rc=$?
else
  timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29733 \
      bench.py --config $C --gpus $N --steps $S --warmup 3 --skip-cpu > gpurun_out/r02_${C}_n$N.log 2>&1; echo $C N=$N rc=$?
fi
grep '^{' gpurun_out/r02_${C}_n$N.log > gpurun_out/r02_${C}_n$N.json || grep -v "^frame\|^ *\^" gpurun_out/r02_${C}_n$N.log | tail -25
python scripts/line_summary.py gpurun_out/r02_${C}_n$N.json
