cd $GRAFT_REPO_ROOT
python -m pytest tests/ -m gpu -x -q -k "int4" 2>&1 | tail -2
for s in "4096 3072 9216" "4608 15360 3072" "4096 1152 3456"; do
  SVDQ_FMT=int4 python tools/time_k2.py $s
done
for v in 3 4; do SVDQ_FMT=int4 SVDQ_LIB=_build_exp/libsvdq_i4e$v.so python tools/time_k2.py 4096 3072 9216 | sed "s/^/e$v /"; done
