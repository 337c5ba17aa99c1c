# HR_OPT_LAZY_RESET: parity, then the bench step with and without it.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_online.py -x -q > $O/gpu_tests_lazy.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_lazy.log
for o in 0 8192 0 8192; do
  echo "$o $(timeout 600 python bench.py --options $o --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/lazy.err)" >> $O/lazy.txt
done
echo "s0/8 $(timeout 600 python bench.py --emulate-shard 0/8 --options 8192 --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/lazy.err)" >> $O/lazy.txt
echo "s0/8base $(timeout 600 python bench.py --emulate-shard 0/8 --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/lazy.err)" >> $O/lazy.txt
HR_OPTS=8192 timeout 900 python scripts/bench_configs.py c4 c2 > $O/lazy_c4.jsonl 2>&1
tail -2 $O/gpu_tests_lazy.log
