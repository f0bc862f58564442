mkdir -p gpurun_out
T=${TAG:-r2ah}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 400 python -m pytest tests -m gpu -q -x -k "eval or rosen or c3" > gpurun_out/${T}_t1.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_t1.log
b() { timeout 200 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline > /tmp/o.log 2>&1; echo "$1: $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"; }
b base
for d in 2 8 16 32; do ES_ASK_DPT=$d b "ask_dpt=$d"; done
for e in 11 16 32 43 64 128; do ES_TELL_ECHUNK=$e b "tell_ec=$e"; done
