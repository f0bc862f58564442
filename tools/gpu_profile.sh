#!/bin/bash
# One gpurun call: bench (default c2), reference arm, ncu launch list, ncu --set full of the hot kernels.
# usage: bash tools/gpu_profile.sh <tag> [bench args...]
TAG=${1:-r01}; shift
OUT=gpurun_out
mkdir -p $OUT
python bench.py "$@" > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"
tail -1 $OUT/bench_$TAG.log
python bench.py --impl reference --steps 5 --warmup 3 "$@" > $OUT/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline $@"
if $CMD > $OUT/plain_$TAG.log 2>&1; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
  KRE=${KRE:-"tell_kernel|ask_kernel|eval_warp|rank_kernel|mlp_kernel|ask_eval_kernel"}
  KCNT=${KCNT:-8}
  ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 8 -c $KCNT -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
else
  echo "plain run failed"; tail -20 $OUT/plain_$TAG.log
fi
