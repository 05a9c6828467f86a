# ncu --set full of one mid-walk level of the narrow D&C walk kernel (W_{4,5})
cd $GRAFT_REPO_ROOT
OUT=gpurun_out; TAG=${1:-pw}
ncu --set full --clock-control none --import-source on -k regex:k_walk_dc -s 14 -c 1 -o $OUT/prof_walk_w45_$TAG python tools/walk_runs.py w45 > $OUT/prof_walk_w45_$TAG.log 2>&1
tail -2 $OUT/prof_walk_w45_$TAG.log | cut -c1-200
