O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 600 python scripts/bench_configs.py c1 c3 > $O/configs_c13.jsonl 2> $O/configs_c13.err
timeout 600 python scripts/smem32_bench.py > $O/smem32.json 2> $O/smem32.err
timeout 900 python bench.py > $O/bench_head.json 2> $O/bench_head.err
tail -2 $O/gpu_tests.log
