O=gpurun_out; mkdir -p $O
python -c "from paper_2401_04701_b200 import build as b; b.build(force=True, extra=['-DHR_CMP_MINB=2'])"
for cfg in "0/8 3 0 x" "0/8 3 256 0" "7/8 3 256 0" "0/2 3 0 x" "0/2 3 256 0"; do
  set -- $cfg
  n=$(echo $1 | tr / _)_g$2_o$3_s$4
  if [ "$4" = x ]; then unset HR_SPLIT_LOG2; else export HR_SPLIT_LOG2=$4; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hr_ --csv \
    --log-file $O/cm_$n.csv python scripts/prof_replay.py --lb 16 --reps 2 --format u64 --shard $1 --granule $2 --options $3 > $O/cm_$n.log 2>&1
done
