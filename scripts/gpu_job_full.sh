# Full check at HEAD: GPU tests, the bench line, emulated shard steps (all ranks
# of N = 2, 4, 8), per-config replay throughput.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
HR_BENCH_STEPLOG=1 timeout 900 python bench.py > $O/bench_head.json 2> $O/bench_head.err
rm -f $O/shards_all.txt
for s in 0/8 1/8 2/8 3/8 4/8 5/8 6/8 7/8 0/4 1/4 2/4 3/4 0/2 1/2; do
  echo "$s $(timeout 300 python bench.py --emulate-shard $s --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/shards_all.err)" >> $O/shards_all.txt
done
echo "1/1 $(timeout 300 python bench.py --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/shards_all.err)" >> $O/shards_all.txt
tail -2 $O/gpu_tests.log
