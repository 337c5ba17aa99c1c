O=gpurun_out; mkdir -p $O; rm -f $O/gsweep.txt
for g in 0 5 9; do
  for r in 0 1 2 3 4 5 6 7; do
    echo "$g $r $(timeout 300 python bench.py --emulate-shard $r/8 --granule-log2 $g --no-e2e --no-cpu --no-slowdown --steps 15 2>/dev/null)" >> $O/gsweep.txt
  done
done
