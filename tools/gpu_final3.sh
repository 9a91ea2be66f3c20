# Round-2 closing evidence with the final build
mkdir -p gpurun_out/final3
python bench.py > gpurun_out/final3/bench_flux.json 2> gpurun_out/final3/bench_flux.err; echo "bench rc=$?"
python bench.py --config pixart --no-cpu-baseline > gpurun_out/final3/bench_pixart.json 2>/dev/null
python bench.py --config sdxl --no-cpu-baseline > gpurun_out/final3/bench_sdxl.json 2>/dev/null
python bench.py --fmt w8a8 --no-cpu-baseline > gpurun_out/final3/bench_flux_w8a8.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final3/bench_ref.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final3/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/final3/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/final3/step_full -f \
    python tools/step_once.py --warm 2 > gpurun_out/final3/step_full.log 2>&1
tail -1 gpurun_out/final3/step_full.log
python - <<'PY'
import json
for c in ("flux", "pixart", "sdxl", "flux_w8a8"):
    d = json.load(open(f"gpurun_out/final3/bench_{c}.json"))
    print(c, d["ms_per_step"], "K2", d["roofline"]["achieved"], d["roofline"]["frac"], "K1", d["k1"]["achieved"], d["k1"]["frac"],
          "lr", (d.get("lowrank_overhead") or {}).get("value"), "e2e", d["e2e"]["value"], d["clocks"])
PY
