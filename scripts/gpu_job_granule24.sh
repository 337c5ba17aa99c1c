# Shard-owner parity, then emulated N = 2 / 4 shard steps per granule (all ranks).
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/gpu_tests_g.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_g.log
for g in 9 3 0; do
  for s in 0/2 1/2 0/4 1/4 2/4 3/4; do
    echo "$g $s $(timeout 300 python bench.py --emulate-shard $s --granule-log2 $g --no-e2e --no-cpu --no-slowdown --steps 3 --warmup 3 2>>$O/gran24.err)" >> $O/gran24.txt
  done
done
tail -2 $O/gpu_tests_g.log
