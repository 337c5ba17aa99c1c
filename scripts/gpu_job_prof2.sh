# ncu --set full at HEAD: the N = 8 address-shard replay (rank 0) and the C3 SMEM-shadow replay.
O=gpurun_out; mkdir -p $O
timeout 1200 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:hr_replay -s 1 -c 1 \
  -o $O/prof_shard0_8_head python scripts/prof_replay.py --lb 16 --reps 2 --format u64 --shard 0/8 --granule 3 > $O/prof_shard_head.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hr_replay -s 1 -c 1 \
  -o $O/prof_c3_head python scripts/prof_config.py c3 > $O/prof_c3_head.log 2>&1
tail -1 $O/prof_shard_head.log; tail -1 $O/prof_c3_head.log
