set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "eval or tell or rastrigin or config2 or config3 or variants or sharded or parity" > gpurun_out/r2a_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r2a_tests.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/r2a_bench.log | cut -c1-600
ncu --set full --clock-control none --import-source on -k regex:"tell_kernel|eval_warp" -s 4 -c 4 -o gpurun_out/r2a_prof python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_ncu.log 2>&1; echo ncu rc=$?
