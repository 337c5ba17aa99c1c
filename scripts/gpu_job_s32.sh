O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "smem32 or ablations" > $O/gpu_tests_s32.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests_s32.log
timeout 600 python scripts/smem32_bench.py > $O/smem32.json 2> $O/smem32.err
STEPS=10 timeout 300 python scripts/step_parts.py 16 > $O/step_parts_plain.txt 2>&1
nvidia-smi --query-gpu=clocks.sm --format=csv -lms 100 > /dev/null 2>&1 &
SMI=$!
STEPS=10 timeout 300 python scripts/step_parts.py 16 > $O/step_parts_smi.txt 2>&1
kill $SMI
timeout 900 python bench.py > $O/bench_head2.json 2> $O/bench_head2.err
tail -2 $O/gpu_tests_s32.log
