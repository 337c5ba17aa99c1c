# Full check at HEAD: GPU tests, smoke, the bench line, emulated shard steps
# (all ranks of N = 2, 4, 8 and the N = 1 step), per-config replay throughput.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_head.json 2> $O/bench_head.err
rm -f $O/shards_all.txt
for s in 0/8 1/8 2/8 3/8 4/8 5/8 6/8 7/8 0/4 1/4 2/4 3/4 0/2 1/2; do
  echo "$s $(timeout 300 python bench.py --emulate-shard $s --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/shards_all.err)" >> $O/shards_all.txt
done
echo "1/1 $(timeout 300 python bench.py --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/shards_all.err)" >> $O/shards_all.txt
timeout 1200 python scripts/bench_configs.py c1 c2 c3 c4 c5 > $O/configs_head.jsonl 2> $O/configs_head.err
tail -2 $O/gpu_tests.log; tail -1 $O/smoke.log
