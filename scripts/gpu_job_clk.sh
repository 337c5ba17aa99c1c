O=gpurun_out; mkdir -p $O; rm -f $O/clk.txt $O/clk.err
for r in 1 2 3 4 5 6; do
  echo "x $(HR_REPORT_PROFILE=1 HR_BENCH_STEPLOG=1 timeout 600 python bench.py --no-e2e --no-cpu --no-slowdown --steps 15 2>>$O/clk.err)" >> $O/clk.txt
done
