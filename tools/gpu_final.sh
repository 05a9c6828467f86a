# round-end evidence: smoke, bench (both arms), big walks with the current walk kernel
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-fin}
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc $?"; tail -1 $OUT/smoke_$TAG.log
python bench.py > $OUT/bench_c5_$TAG.log 2>&1; tail -1 $OUT/bench_c5_$TAG.log | cut -c1-200
python bench.py --impl reference > $OUT/bench_ref_$TAG.log 2>&1; tail -1 $OUT/bench_ref_$TAG.log | cut -c1-200
export BDEG_DEBUG=1 BDEG_DEBUG_LEVELS=1
timeout 1200 python tools/walk_runs.py w46 > $OUT/walk_w46_$TAG.log 2>&1; echo "w46 rc $?"; tail -1 $OUT/walk_w46_$TAG.log | cut -c1-250
timeout 1500 python tools/walk_runs.py w55 > $OUT/walk_w55_$TAG.log 2>&1; echo "w55 rc $?"; tail -1 $OUT/walk_w55_$TAG.log | cut -c1-250
