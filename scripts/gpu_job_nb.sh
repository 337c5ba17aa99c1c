O=gpurun_out; mkdir -p $O; rm -f $O/nb.txt
for nb in 2 3 4; do
  python -c "from paper_2401_04701_b200 import build as b; b.build(force=True, extra=['-DHR_STAGE_NB_ROW=$nb'])" > /dev/null 2>&1
  for s in 1/1 0/8; do
    if [ $s = 1/1 ]; then a=""; else a="--emulate-shard $s"; fi
    echo "$nb $s $(timeout 300 python bench.py $a --no-e2e --no-cpu --no-slowdown --steps 15 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"ms_per_step\"],2), round(d[\"step_breakdown_ms\"][\"replay_kernel\"],2), d[\"parity_vs_closed_form\"])")" >> $O/nb.txt
  done
done
cat $O/nb.txt
