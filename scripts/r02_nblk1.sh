# nblk = 1 at N > 1 (no forward sweep) where HBM allows: c2 at N=4 / N=2, c4 at N=4
run() {  # config N
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 2975$2 \
      bench.py --config $1 --gpus $2 --steps 3 --warmup 3 --skip-cpu --nblk 1 > gpurun_out/nb1_$1_n$2.log 2>&1; echo $1 N=$2 rc=$?
  grep '^{' gpurun_out/nb1_$1_n$2.log > gpurun_out/nb1_$1_n$2.json && python scripts/line_summary.py gpurun_out/nb1_$1_n$2.json | head -1
  grep -i "out of memory\|Error" gpurun_out/nb1_$1_n$2.log | head -3
}
run c2 4
CUDA_VISIBLE_DEVICES=0,1 run c2 2
run c4 4
