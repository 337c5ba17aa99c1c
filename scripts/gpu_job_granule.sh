# Parity of the rotated-stripe shard owner, then emulated N = 8 shard steps per granule.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > $O/gpu_tests_g.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_g.log
for g in 9 5 3 0; do
  for r in 0 1 2 3 4 5 6 7; do
    timeout 300 python bench.py --emulate-shard $r/8 --granule-log2 $g --no-e2e --no-cpu --no-slowdown --steps 3 --warmup 3 >> $O/gran.jsonl 2>>$O/gran.err
  done
done
tail -2 $O/gpu_tests_g.log
