# bench lines for every config + the K2 tests (default tile) + the 384 opt-in test
mkdir -p gpurun_out
python -m pytest tests/test_gpu_k2.py -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench_flux.json 2> gpurun_out/bench_flux.err
python bench.py --config pixart --no-cpu-baseline > gpurun_out/bench_pixart.json 2> gpurun_out/bench_pixart.err
python bench.py --config sdxl --no-cpu-baseline > gpurun_out/bench_sdxl.json 2> gpurun_out/bench_sdxl.err
for c in flux pixart sdxl; do python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.load(open(f"gpurun_out/bench_{c}.json"))
lo = d.get("lowrank_overhead") or {}
print(c, d["ms_per_step"], "K2 frac", d["roofline"]["frac"], "K1 frac", d["k1"]["frac"], "lowrank", lo.get("value"), lo.get("per_launch"))
print("  ", [(l["layers"][0], l["k1_us"], l["k2_us"]) for l in d["per_launch"]])
PY
done
