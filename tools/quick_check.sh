# quick GPU check after a kernel change: math + parity tests, then a short C4 bench line
# usage: bash tools/quick_check.sh TAG [pytest-args...]
TAG=${1:-q}; shift
timeout 600 python -m pytest tests/test_gpu_p2p_math.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q "$@" > gpurun_out/${TAG}_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
d = json.load(open(f"gpurun_out/{t}_bench.json"))
print("ms/step", round(d["ms_per_step"], 3), "value", f'{d["value"]:.4g}', "P2P frac", d["roofline"]["frac"], "M2L frac", d["roofline_m2l"]["frac"])
for k, v in d["config"]["per_tiling"].items():
    print(k, {a: round(b, 3) for a, b in v.items() if a.endswith("ms")})
PY
