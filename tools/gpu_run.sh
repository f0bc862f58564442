#!/bin/bash
# One gpurun call driven by env vars (everything lands in gpurun_out/<TAG>_*):
#   TESTS="-k expr"  pytest -m gpu selection ("" = skip, "all" = the whole suite)
#   BENCH="args;args" bench.py invocations (";"-separated), each logged
#   NCU_K=regex NCU_C=count NCU_ARGS="bench args": one ncu --set full capture of those kernels
#   LAUNCH="bench args" ncu launch list (gpu__time_duration) of one bench invocation
# usage: TAG=r2b TESTS="-k mlp" BENCH="--config c4" bash tools/gpu_run.sh
TAG=${TAG:-r2}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${TAG}_build.log 2>&1 || { echo build failed; tail -20 $OUT/${TAG}_build.log; exit 1; }
if [ -n "$TESTS" ]; then
  if [ "$TESTS" = "all" ]; then SEL=""; else SEL="$TESTS"; fi
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q --maxfail=25 $SEL > $OUT/${TAG}_tests.log 2>&1
  echo "tests rc=$?"; tail -4 $OUT/${TAG}_tests.log
fi
if [ -n "$BENCH" ]; then
  IFS=';' read -ra BS <<< "$BENCH"
  i=0
  for b in "${BS[@]}"; do
    timeout 900 python bench.py $b > $OUT/${TAG}_bench$i.log 2>&1
    echo "bench[$i] ($b) rc=$?"; tail -1 $OUT/${TAG}_bench$i.log | cut -c1-1500
    i=$((i+1))
  done
fi
if [ -n "$LAUNCH" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py $LAUNCH --no-cpu-baseline > $OUT/${TAG}_launch.log 2>&1
  echo "launch list rc=$?"
fi
if [ -n "$NCU_K" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c ${NCU_C:-4} \
    -o $OUT/${TAG}_prof python bench.py $NCU_ARGS --no-cpu-baseline > $OUT/${TAG}_ncu.log 2>&1
  echo "ncu rc=$?"; tail -3 $OUT/${TAG}_ncu.log
fi
