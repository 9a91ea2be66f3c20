# L2 banding: correctness (bitwise vs unbanded) + C5 stack A/B
python -m pytest tests/test_gpu_k2_band.py tests/test_gpu_k2.py tests/test_gpu_step_full.py -x -q 2>&1 | tail -2
SVDQ_K2_BAND_MB=0 python tools/c5_stack.py --out gpurun_out/c5_noband.json 2>&1 | grep C5
python tools/c5_stack.py 2>&1 | grep C5
