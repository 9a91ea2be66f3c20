# One GPU pass: default bench line, ncu launch list of a bench run, ncu --set full of the step's
# 12 launches (grouped FLUX step), CPU-free.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/step_full -f \
    python tools/step_once.py --warm 2 > gpurun_out/step_full.log 2>&1
tail -3 gpurun_out/step_full.log
cat gpurun_out/bench.json
