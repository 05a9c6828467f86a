# profiles of the current kernel: launch list + ncu --set full of C5 and W_{2,4}; A/B of scratch libs
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-prof}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_c5_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_w26_$TAG python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for lib in scratch/libbdeg_mb5.so; do
  for i in 1 2; do
    BDEG_LIB=$lib python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c100-190
    python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c100-190
  done
done
ls $OUT
export BDEG_DEBUG=1 BDEG_DEBUG_LEVELS=1
WALK_SEED=2 timeout 1800 python tools/walk_runs.py w55 > $OUT/walk_w55_seed2.log 2>&1; echo "w55 s2 rc $?"; tail -1 $OUT/walk_w55_seed2.log | cut -c1-300
WALK_SEED=2 timeout 1200 python tools/walk_runs.py w38 > $OUT/walk_w38_seed2.log 2>&1; echo "w38 s2 rc $?"; tail -1 $OUT/walk_w38_seed2.log | cut -c1-300
