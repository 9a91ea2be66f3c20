# ncu evidence for C2 / C3 (launch lists + --set full of the step) and the INT4 K2 (one FLUX step)
mkdir -p gpurun_out
for c in pixart sdxl; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv \
      --profile-from-start off python tools/step_once.py --config $c > gpurun_out/launches_$c.log 2>&1
  ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_$c -f \
      python tools/step_once.py --config $c > gpurun_out/step_$c.log 2>&1
  tail -1 gpurun_out/step_$c.log
done
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k2_int4 -c 2 -o gpurun_out/int4_full -f \
    python tools/step_once.py --fmt int4 > gpurun_out/int4_full.log 2>&1
tail -1 gpurun_out/int4_full.log
