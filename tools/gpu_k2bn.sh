set -x
python -m pytest tests/test_gpu_k2.py tests/test_gpu_step_full.py tests/test_gpu_configs.py -x -q 2>&1 | tail -5
for s in "4608 3072 21504" "4096 3072 9216" "4608 15360 3072" "4096 3072 3072" "4096 3072 12288" "4096 12288 3072" "512 3072 9216" "512 3072 3072"; do
  python tools/time_k2.py $s
  SVDQ_K2_BN=192 python tools/time_k2.py $s | sed 's/^/bn192 /'
done
python bench.py --no-cpu-baseline > gpurun_out/bench_bn256.json 2> gpurun_out/bench_bn256.err
SVDQ_K2_BN=192 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench_bn192.json 2>> gpurun_out/bench_bn256.err
python -c "
import json
for n in ('bn256','bn192'):
  d=json.load(open('gpurun_out/bench_%s.json'%n)); print(n, d['ms_per_step'], d['roofline']['achieved'], [ (l['layers'][0], l['k1_us'], l['k2_us']) for l in d['per_launch']])
"
