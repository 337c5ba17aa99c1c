O=gpurun_out; mkdir -p $O; rm -f $O/async.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "report_async or lazy or smem32 or shard" > $O/gpu_tests_async.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_async.log
for r in 1 2 3 4; do
  echo "async $(timeout 600 python bench.py --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/async.err)" >> $O/async.txt
done
echo "sync $(timeout 600 python bench.py --sync-report --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/async.err)" >> $O/async.txt
tail -2 $O/gpu_tests_async.log
