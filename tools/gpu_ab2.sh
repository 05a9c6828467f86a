# A/B: numerator-bound checks in the enumeration elimination (new lib vs scratch/libbdeg_base.so),
# narrow (int32) vs int64 D&C walk; then the GPU test suite
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-ab2}
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"; tail -3 $OUT/pytest_gpu_$TAG.log
for i in 1 2; do
python bench.py --no-cpu-baseline > $OUT/bench_c5_new${i}_$TAG.log 2>&1; tail -1 $OUT/bench_c5_new${i}_$TAG.log | cut -c100-200
BDEG_LIB=scratch/libbdeg_base.so python bench.py --no-cpu-baseline > $OUT/bench_c5_base${i}_$TAG.log 2>&1; tail -1 $OUT/bench_c5_base${i}_$TAG.log | cut -c100-200
done
for wl in w24 w25 w26; do
python bench.py --workload $wl --steps 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200
BDEG_LIB=scratch/libbdeg_base.so python bench.py --workload $wl --steps 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200
done
export BDEG_DEBUG=1
timeout 300 python tools/walk_runs.py w36,w45,w37 > $OUT/walk_narrow_$TAG.log 2>&1; grep '^{' $OUT/walk_narrow_$TAG.log | cut -c1-200; grep narrow $OUT/walk_narrow_$TAG.log | cut -c1-250
BDEG_WALK_WIDE=1 timeout 300 python tools/walk_runs.py w36,w45,w37 > $OUT/walk_wide_$TAG.log 2>&1; grep '^{' $OUT/walk_wide_$TAG.log | cut -c1-200
