set -x
python -m pytest tests/test_gpu_k1.py tests/test_gpu_step_full.py tests/test_gpu_tp.py tests/test_gpu_configs.py -x -q 2>&1 | tail -4
for s in "4608 3072" "4608 15360" "4608 12288" "512 3072" "4096 1152"; do python tools/time_k1.py $s; done
bash tools/trace_k1.sh > /dev/null 2>&1
for s in "4608 3072" "4608 15360"; do
  SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s
done
python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench_k1v3.json 2> gpurun_out/bench_k1v3.err
python -c "
import json
d=json.load(open('gpurun_out/bench_k1v3.json')); print(d['ms_per_step'], d['roofline']['frac'], d['k1'], [(l['k1_us'], l['k2_us']) for l in d['per_launch']])"
