O=gpurun_out; mkdir -p $O
timeout 1500 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:hr_replay -s 1 -c 1 \
  -o $O/prof_replay_c32 python scripts/prof_replay.py --lb 16 --reps 2 --format c32 > $O/prof_replay_c32.log 2>&1
timeout 900 python bench.py > $O/bench_c32.json 2> $O/bench_c32.err
tail -1 $O/prof_replay_c32.log
