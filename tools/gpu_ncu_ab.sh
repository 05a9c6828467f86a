# ncu --set full of the C5 enumeration kernel with and without certificate pruning
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-ab}
ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_c5_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
BDEG_NO_CERT=1 ncu --set full --clock-control none --import-source on -k regex:k_enumerate -s 6 -c 1 -o $OUT/prof_c5_nocert_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls $OUT
