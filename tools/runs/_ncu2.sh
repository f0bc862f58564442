mkdir -p gpurun_out
T=${TAG:-r2s}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mlp32_kernel" -s 1 -c 1 -o gpurun_out/${T}_mlp32 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu32.log 2>&1; echo ncu32 rc=$?
timeout 300 python bench.py --config c4 --mlp fp16 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain16.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mlp_kernel" -s 1 -c 1 -o gpurun_out/${T}_mlp16 python bench.py --config c4 --mlp fp16 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu16.log 2>&1; echo ncu16 rc=$?
