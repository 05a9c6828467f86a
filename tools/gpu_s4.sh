cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-s4}
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; rc=$?; echo "pytest rc $rc"; tail -3 $OUT/pytest_gpu_$TAG.log
[ $rc -ne 0 ] && exit 1
python bench.py > $OUT/bench_c5_$TAG.log 2>&1; tail -1 $OUT/bench_c5_$TAG.log | cut -c1-300
python bench.py --workload w26 --steps 3 --no-cpu-baseline > $OUT/bench_w26_$TAG.log 2>&1; tail -1 $OUT/bench_w26_$TAG.log | cut -c1-200
export BDEG_DEBUG=1
timeout 300 python tools/walk_runs.py w44,w28,w36,w45,w37 > $OUT/walk_$TAG.log 2>&1; grep '^{' $OUT/walk_$TAG.log | cut -c1-160; grep narrow $OUT/walk_$TAG.log | cut -c1-250
BDEG_DEBUG_LEVELS=1 timeout 2400 python tools/walk_runs.py w55 > $OUT/walk_w55_$TAG.log 2>&1; echo "w55 rc $?"; tail -2 $OUT/walk_w55_$TAG.log | cut -c1-400
