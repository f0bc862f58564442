mkdir -p gpurun_out
T=${TAG:-r2final5}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gpu_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_gpu_tests.log; grep -E "^FAILED" gpurun_out/${T}_gpu_tests.log | head
bash tools/runs/_final2.sh
