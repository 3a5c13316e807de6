#!/bin/bash
# A/B the multi-point CG: alternate library builds, 3 runs each (cfg4 slice)
#   tools/ab_multi.sh A.so B.so [n_pts] [iters]
N=${3:-2368}; I=${4:-400}
for r in 1 2 3; do
  for L in "$1" "$2"; do
    MFB_ALLOW_FOREIGN_LIBRARY=1 MFB_LIBRARY=$L timeout 300 python tools/prof_cg_multi.py $N $I multi 2>&1 | tail -1 | sed "s|^|$(basename $L) |"
  done
done
