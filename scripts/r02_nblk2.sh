# fewer checkpoint blocks where HBM allows: c4 at N=2 (nblk 2), c5 at N=4 (nblk 4)
run() {  # config N nblk
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 2976$2 \
      bench.py --config $1 --gpus $2 --steps 2 --warmup 3 --skip-cpu --nblk $3 > gpurun_out/nb_$1_n$2_b$3.log 2>&1; echo $1 N=$2 nblk=$3 rc=$?
  grep '^{' gpurun_out/nb_$1_n$2_b$3.log > gpurun_out/nb_$1_n$2_b$3.json
  python scripts/line_summary.py gpurun_out/nb_$1_n$2_b$3.json 2>/dev/null | head -1
  grep -i "out of memory" gpurun_out/nb_$1_n$2_b$3.log | head -2
}
CUDA_VISIBLE_DEVICES=0,1 run c4 2 2
run c5 4 4
