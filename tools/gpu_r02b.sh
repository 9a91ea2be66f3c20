# planner check + full GPU tests + bench lines (all configs)
mkdir -p gpurun_out
python tools/k2_shape_sweep.py planner > gpurun_out/k2plan.log 2>&1
SVDQ_K2_PAIR=1 python tools/k2_shape_sweep.py pair >> gpurun_out/k2plan.log 2>&1
cat gpurun_out/k2plan.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_flux.json 2> gpurun_out/bench_flux.err; echo "bench rc=$?"
python bench.py --config pixart --no-cpu-baseline > gpurun_out/bench_pixart.json 2> gpurun_out/bench_pixart.err
python bench.py --config sdxl --no-cpu-baseline > gpurun_out/bench_sdxl.json 2> gpurun_out/bench_sdxl.err
for c in flux pixart sdxl; do python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.load(open(f"gpurun_out/bench_{c}.json"))
lo = d.get("lowrank_overhead") or {}
print(c, d["ms_per_step"], "K2 frac", d["roofline"]["frac"], "K1 frac", d["k1"]["frac"], "lowrank", lo.get("value"))
print("  ", [(l["layers"][0], l["k1_us"], l["k2_us"]) for l in d["per_launch"]])
PY
done
