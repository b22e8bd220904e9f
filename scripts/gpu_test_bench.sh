#!/bin/bash
# One gpurun call: GPU parity tests, then the default bench (softmax) and the QLA bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
python bench.py --attn qla --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_qla.json 2> gpurun_out/bench_qla.err; echo qla_exit=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench.json", "gpurun_out/bench_qla.json"):
    try:
        d = json.load(open(f))
        r = d["roofline"]
        print(f, "value=%.4g" % d["value"], "ms/step=%.4f" % d["ms_per_step"], "kernel_ms=", r["kernel_ms"],
              "frac=", r["frac"], r["bound"], "clocks=", d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
tail -3 gpurun_out/bench.err
