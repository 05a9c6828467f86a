# final evidence for the current kernel: tests, smoke, bench (both arms), launch list, ncu --set full
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-f2}
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"; tail -1 $OUT/pytest_gpu_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc $?"
python bench.py > $OUT/bench_c5_$TAG.log 2>&1; tail -1 $OUT/bench_c5_$TAG.log | cut -c1-200
python bench.py --impl reference --steps 10 --warmup 3 > $OUT/bench_ref_$TAG.log 2>&1; tail -1 $OUT/bench_ref_$TAG.log | cut -c1-200
python bench.py --workload w26 --steps 3 --no-cpu-baseline > $OUT/bench_w26_$TAG.log 2>&1; tail -1 $OUT/bench_w26_$TAG.log | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_c5_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_w26_$TAG python bench.py --workload w26 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls $OUT | grep $TAG
