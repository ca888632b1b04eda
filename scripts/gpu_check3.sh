mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "tcgen05 or tensor_cores or hub" > gpurun_out/pytest_tc.log 2>&1; echo tc-tests rc=$?
tail -15 gpurun_out/pytest_tc.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench_tc.log 2>&1; echo bench rc=$?
python - <<'PY'
import json
l=[x for x in open("gpurun_out/bench_tc.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("ms/step", d["ms_per_step"], "value", d["value"], "e2e", d["e2e"] and d["e2e"]["ms_per_step"])
    for k,v in list(d["kernels"].items())[:8]: print(k, round(v["ms_total"],1), v["launches"])
else:
    print(open("gpurun_out/bench_tc.log").read()[-3000:])
PY
