mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -20
grep -B2 "AssertionError" gpurun_out/pytest_gpu.log | grep "^E" | head -20
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench_tc.log 2>&1; echo bench rc=$?
python - <<'PY'
import json
l=[x for x in open("gpurun_out/bench_tc.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("ms/step", d["ms_per_step"], "value", d["value"], "e2e", d["e2e"] and d["e2e"]["ms_per_step"], "loss", d["loss"])
    for k,v in list(d["kernels"].items())[:12]: print(k, round(v["ms_total"]/d["steps"],1), v["launches"]//d["steps"])
    print(json.dumps(d["roofline"])); print(json.dumps(d["spmm_roofline"]))
else:
    print(open("gpurun_out/bench_tc.log").read()[-3000:])
PY
