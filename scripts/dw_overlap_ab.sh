# weight gradient on a side stream: engine tests, then c2 N=1 with and without the overlap
timeout 900 python -m pytest tests/test_gpu_engine.py -q -m gpu -x 2>&1 | tail -2
for ov in 1 0 1; do
  DGNN_DW_OVERLAP=$ov timeout 900 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/ov$ov.log 2>&1
  echo "overlap=$ov $(grep '^{' gpurun_out/ov$ov.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"])')"
done
