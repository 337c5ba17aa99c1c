O=gpurun_out; mkdir -p $O; rm -f $O/shards_final.txt
for s in 0/8 1/8 2/8 3/8 4/8 5/8 6/8 7/8 0/4 1/4 2/4 3/4 0/2 1/2; do
  echo "$s $(timeout 300 python bench.py --emulate-shard $s --no-e2e --no-cpu --no-slowdown --steps 15 2>/dev/null)" >> $O/shards_final.txt
done
echo "1/1 $(timeout 300 python bench.py --no-e2e --no-cpu --no-slowdown --steps 15 2>/dev/null)" >> $O/shards_final.txt
