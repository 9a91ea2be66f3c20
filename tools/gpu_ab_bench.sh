# A/B of the FLUX bench step: current lib vs _build_exp/libsvdq_nopipe.so (pre-team K1, pre-planner K2), alternating
for i in 1 2; do
  for v in new old; do
    if [ "$v" = new ]; then L=""; else L=_build_exp/libsvdq_nopipe.so; fi
    SVDQ_LIB=$L python bench.py --no-cpu-baseline > gpurun_out/ab_$v$i.json 2>/dev/null
    python - "$v" gpurun_out/ab_$v$i.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
print(sys.argv[1], d["ms_per_step"], "K2", d["roofline"]["achieved"], "K1", d["k1"]["achieved"],
      [(l["layers"][0][:12], l["k1_us"], l["k2_us"]) for l in d["per_launch"]])
PY
  done
done
