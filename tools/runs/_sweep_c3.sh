python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { timeout 120 env "$@" python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'; }
echo base; run X=1
for e in 8 12 16 32 43 64; do echo "echunk $e"; run ES_TELL_ECHUNK=$e; done
for d in 4 8 16 32; do echo "dpt $d"; run ES_ASK_DPT=$d; done
