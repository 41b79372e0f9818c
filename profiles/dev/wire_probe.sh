# A/B of the host-flavour output wire (16-bit vs 32-bit) through bench.py's e2e pass.
timeout 300 python -m pytest tests/test_host_pipeline_gpu.py -q -x 2>&1 | tail -2
for w in 16 32; do
  if [ $w = 32 ]; then export BITMM_HOST_WIRE=32; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_wire$w.json 2>&1
  W=$w python - <<'PY'
import json, os
d = json.load(open(f"gpurun_out/bench_wire{os.environ['W']}.json"))
e = d["e2e"]
print(os.environ["W"], round(d["value"]), round(e["value"], 2), round(e["ms_per_step"], 3), {k: round(v, 3) for k, v in e["ms_per_call"].items()})
PY
done
unset BITMM_HOST_WIRE
BITMM_WIRE_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>&1 >/dev/null | grep "bitmm wire" | tail -6
BITMM_HOST_SIMD=sse2 BITMM_WIRE_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>&1 >/dev/null | grep "bitmm wire" | tail -3
