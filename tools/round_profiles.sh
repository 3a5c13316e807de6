#!/bin/bash
# Round profiling pass on the GPU box (one GPU): bench line, ncu launch list of
# the bench command, full captures of the dominant kernels, summaries.
# usage: bash tools/round_profiles.sh <outdir>   (run from the repo root)
set -x
OUT=${1:-gpurun_out/prof}
mkdir -p $OUT
python bench.py > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-s2 \
    > $OUT/ncu_launch.log 2>&1
for k in band_solve cg_pair condense; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $OUT/$k \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-s2 > $OUT/ncu_$k.log 2>&1
  python tools/ncu_summary.py $OUT/$k.ncu-rep $OUT/${k}_cfg2_summary.json > /dev/null
  ncu -i $OUT/$k.ncu-rep --page source --csv --print-source=cuda,sass > $OUT/${k}_src.csv 2>/dev/null
  python tools/ncu_lines.py $OUT/${k}_src.csv 15 > $OUT/${k}_cfg2_hotlines.txt
done
ncu --set full --import-source on --clock-control none -k regex:cg_multi -c 1 -o $OUT/cg_multi \
    python tools/prof_cg_multi.py 1184 100 multi > $OUT/ncu_cg_multi.log 2>&1
python tools/ncu_summary.py $OUT/cg_multi.ncu-rep $OUT/cg_multi_cfg4_summary.json > /dev/null
ncu -i $OUT/cg_multi.ncu-rep --page source --csv --print-source=cuda,sass > $OUT/cg_multi_src.csv 2>/dev/null
python tools/ncu_lines.py $OUT/cg_multi_src.csv 15 > $OUT/cg_multi_cfg4_hotlines.txt
for c in cfg1 cfg2 cfg3; do python tools/phase_timing.py $c >> $OUT/phase_timing.txt 2>&1; done
for c in cfg1 cfg2; do python tools/phase_timing.py $c --method S2 >> $OUT/phase_timing_s2.txt 2>&1; done
python tools/basis_bench.py cfg4 >> $OUT/phase_timing.txt 2>&1
python tools/basis_bench.py cfg5 >> $OUT/phase_timing.txt 2>&1
python tools/prof_cg_multi.py 1184 200 both >> $OUT/phase_timing.txt 2>&1
rm -f $OUT/*_src.csv
