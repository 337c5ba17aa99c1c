# GPU parity + address-shard timings of the pooled kernel (N = 8 projection).
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
for s in 0/8 7/8; do
  n=$(echo $s | tr / _)
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hr_replay --csv \
    --log-file $O/pl_$n.csv python scripts/prof_replay.py --lb 16 --reps 2 --format u64 --shard $s > $O/pl_$n.log 2>&1
done
for s in 0/8 7/8 0/4 0/2; do
  timeout 600 python bench.py --emulate-shard $s --no-e2e --no-cpu --no-slowdown >> $O/shards.jsonl 2>>$O/shards.err
done
tail -2 $O/gpu_tests.log
