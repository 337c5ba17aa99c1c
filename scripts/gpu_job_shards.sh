set -x
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_atomics.cu 2>/dev/null
timeout 300 /tmp/mb 0 big > $O/mb_g0.txt 2>&1
timeout 300 /tmp/mb 32 big > $O/mb_g32.txt 2>&1
timeout 300 /tmp/mb 128 big > $O/mb_g128.txt 2>&1
for s in 0/2 1/2 0/4 3/4 0/8 7/8; do
  timeout 600 python bench.py --emulate-shard $s --no-e2e --no-cpu --no-slowdown --steps 5 --warmup 3 >> $O/shards.jsonl 2>>$O/shards.err
done
for s in 0/8 7/8; do
  n=$(echo $s | tr / _)
  HR_DEBUG_CHOICE=1 timeout 900 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:hr_replay -s 1 -c 1 -o $O/prof_shard_$n python scripts/prof_replay.py --lb 16 --reps 2 --format u64 --shard $s > $O/prof_shard_$n.log 2>&1
done
