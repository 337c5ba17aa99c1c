# End-of-round evidence at HEAD: GPU tests, smoke, bench line, launch list of the bench command.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_final.json 2> $O/bench_final.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-slowdown > $O/launches_final.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
tail -2 $O/gpu_tests.log; tail -1 $O/smoke.log
