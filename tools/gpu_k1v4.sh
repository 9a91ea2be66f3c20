python -m pytest tests/test_gpu_k1.py tests/test_gpu_tp.py tests/test_gpu_step_full.py tests/test_gpu_configs.py tests/test_gpu_w8a8.py -x -q 2>&1 | tail -2
bash tools/gpu_k1abl.sh 2>&1 | grep -v "issue times\|seen by\|L1s issue\|MMA passes"
python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench_k1v4.json 2> gpurun_out/bench_k1v4.err
python -c "
import json
d=json.load(open('gpurun_out/bench_k1v4.json')); print(d['ms_per_step'], d['roofline']['frac'], d['k1']['frac'], d['kernel_sum_ms'], [(l['k1_us'], l['k2_us']) for l in d['per_launch']])"
