mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x -k "weight_grad" > gpurun_out/pytest_dw.log 2>&1; echo dw-tests rc=$?
tail -5 gpurun_out/pytest_dw.log
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench_tc.log 2>&1; echo bench rc=$?
python - <<'PY'
import json
l=[x for x in open("gpurun_out/bench_tc.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("ms/step", d["ms_per_step"], "value", d["value"], "e2e", d["e2e"] and d["e2e"]["ms_per_step"], "loss", d["loss"])
    for k,v in list(d["kernels"].items())[:10]: print(k, round(v["ms_total"]/d["steps"],1), v["launches"]//d["steps"])
else:
    print(open("gpurun_out/bench_tc.log").read()[-3000:])
PY
