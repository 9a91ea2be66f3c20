python tools/k2_shape_sweep.py default
SVDQ_K2_PAIR=0 python tools/k2_shape_sweep.py 1cta
SVDQ_K2_PAIR=0 SVDQ_K2_BN1=128 python tools/k2_shape_sweep.py 1cta128
SVDQ_K2_PAIR=1 python tools/k2_shape_sweep.py pair
SVDQ_K2_PAIR=1 SVDQ_K2_BN=192 python tools/k2_shape_sweep.py pair192
