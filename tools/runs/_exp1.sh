# tell occupancy (minBlocks) x entry-chunk sweep at c2; per-handle tell times
mkdir -p gpurun_out
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
for mb in 8 10 12; do
  cp exp/libes_mb$mb.so paper_2212_04180_b200/lib/libes_b200.so
  for ec in "" 8 13 16 20 26 32 43 64; do
    ES_TELL_ECHUNK=$ec timeout 300 python bench.py --steps 20 --warmup 5 --sub 0 --no-cpu-baseline > /tmp/o.log 2>&1
    echo "mb=$mb ec=$ec $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d["kernel_ms_by_handle"]))' 2>&1)" >> gpurun_out/exp1.txt
  done
  ES_TELL_ECHUNK= timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1
  echo "c5 mb=$mb $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d["kernel_ms_by_handle"]), d["roofline"]["frac"])' 2>&1)" >> gpurun_out/exp1.txt
done
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
