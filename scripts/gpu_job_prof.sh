# Round-1 evidence at HEAD: the bench line, the launch list of the bench command,
# one ncu --set full capture of the replay kernel at full size (C5, N = 1).
O=gpurun_out; mkdir -p $O
timeout 900 python bench.py > $O/bench_final.json 2> $O/bench_final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-slowdown > $O/launches_final.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:hr_replay -s 1 -c 1 \
  -o $O/prof_replay_final python scripts/prof_replay.py --lb 16 --reps 2 --format u64 > $O/prof_replay_final.log 2>&1
tail -2 $O/prof_replay_final.log
