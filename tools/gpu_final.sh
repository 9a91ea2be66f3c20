# Final round-2 evidence: bench lines (all configs + reference arm), launch list + ncu of the FLUX
# step, C5 stack, TP emulation (P = 1, 2, 4, 8 at batch 1 / 8, all-gather and fused gather)
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_flux.json 2> gpurun_out/final/bench_flux.err; echo "bench rc=$?"
python bench.py --config pixart --no-cpu-baseline > gpurun_out/final/bench_pixart.json 2>/dev/null
python bench.py --config sdxl --no-cpu-baseline > gpurun_out/final/bench_sdxl.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/bench_ref.json 2>/dev/null
python tools/c5_stack.py --out gpurun_out/final/c5_stack_1gpu.json 2>&1 | grep C5
for B in 1 8; do for P in 1 2 4 8; do for G in nccl fused; do
  if [ $P = 1 ] && [ $G = fused ]; then continue; fi
  python bench.py --mode tp --tp-emulate $P --batch $B --tp-gather $G --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/final/tp_P${P}_B${B}_$G.json 2>/dev/null
done; done; done
ls gpurun_out/final | wc -l
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/final/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/final/step_full -f \
    python tools/step_once.py --warm 2 > gpurun_out/final/step_full.log 2>&1
tail -1 gpurun_out/final/step_full.log
python - <<'PY'
import json
for c in ("flux", "pixart", "sdxl"):
    d = json.load(open(f"gpurun_out/final/bench_{c}.json"))
    print(c, d["ms_per_step"], "K2", d["roofline"]["achieved"], d["roofline"]["frac"], "K1", d["k1"]["achieved"], d["k1"]["frac"],
          "lr", (d.get("lowrank_overhead") or {}).get("value"), "e2e", d["e2e"]["value"], d["clocks"])
PY
