#!/bin/bash
# Round-2 profiling pass on the GPU box (one GPU): bench line on cfg4, ncu
# launch list of the same command, full capture of the dominant kernel (the
# multi-point CG on a cfg4 slice) and of the Darcy condensation on cfg5, the
# full cfg4 sweep. usage: bash tools/round2_profiles.sh <outdir>
set -x
OUT=${1:-gpurun_out/prof2}
mkdir -p $OUT
python bench.py --steps 6 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches_cfg4_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
    > $OUT/ncu_launch.log 2>&1
python tools/launch_summary.py $OUT/launches_cfg4_bench.csv \
    "ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 python bench.py --steps 1 --warmup 0 --no-cpu-baseline" \
    > $OUT/launches_cfg4_bench_summary.txt
ncu --set full --import-source on --clock-control none -k regex:cg_multi_kernel -c 1 -o $OUT/cg_multi \
    python tools/prof_cg_multi.py 1184 100 multi 23 > $OUT/ncu_cg_multi.log 2>&1
python tools/ncu_summary.py $OUT/cg_multi.ncu-rep $OUT/cg_multi_cfg4_summary.json > /dev/null
ncu -i $OUT/cg_multi.ncu-rep --page source --csv --print-source=cuda,sass > $OUT/cg_multi_src.csv 2>/dev/null
python tools/ncu_lines.py $OUT/cg_multi_src.csv 20 > $OUT/cg_multi_cfg4_hotlines.txt
rm -f $OUT/cg_multi_src.csv
python tools/cfg4_sweep.py --max-iter 200000 --json $OUT/cfg4_sweep.json > $OUT/cfg4_sweep.log 2>&1
python tools/prof_cg_multi.py 6785 0 abs 8 > $OUT/cg_multi_ab.log 2>&1
