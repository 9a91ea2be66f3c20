# Full GPU pass: gpu tests, bench lines for every config, launch list, ncu --set full of the step.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_flux.json 2> gpurun_out/bench_flux.err; echo "bench rc=$?"
python bench.py --config pixart --no-cpu-baseline > gpurun_out/bench_pixart.json 2> gpurun_out/bench_pixart.err
python bench.py --config sdxl --no-cpu-baseline > gpurun_out/bench_sdxl.json 2> gpurun_out/bench_sdxl.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_full -f \
    python tools/step_once.py --warm 2 > gpurun_out/step_full.log 2>&1
tail -2 gpurun_out/step_full.log
for c in flux pixart sdxl; do python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
d = json.load(open(f"gpurun_out/bench_{c}.json"))
lo = d.get("lowrank_overhead") or {}
print(c, d["ms_per_step"], "K2 frac", d["roofline"]["frac"], "K1 frac", d["k1"]["frac"], "lowrank", lo.get("value"))
print("  ", [(l["layers"][0], l["k1_us"], l["k2_us"]) for l in d["per_launch"]])
PY
done
