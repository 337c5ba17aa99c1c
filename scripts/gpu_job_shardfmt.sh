# Launch lists of address-shard replays at N = 8: pooled row kernel vs the
# compacted stream (HR_OPT_POOL_WIDE -> compaction), granule 2^9 vs 2^0.
O=gpurun_out; mkdir -p $O
for cfg in "0/8 9 0" "7/8 9 0" "0/8 9 256" "7/8 9 256" "0/8 0 0" "0/8 0 256" "7/8 0 256" "0/8 5 256"; do
  set -- $cfg
  n=$(echo $1 | tr / _)_g$2_o$3
  HR_DEBUG_CHOICE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hr_ --csv \
    --log-file $O/ll_$n.csv python scripts/prof_replay.py --lb 16 --reps 2 --format u64 --shard $1 --granule $2 --options $3 > $O/ll_$n.log 2>&1
done
