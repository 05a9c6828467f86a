# Table 3 ">=" entries by the cell walk; W_{4,6} again under a second lifting
cd $GRAFT_REPO_ROOT
export BDEG_DEBUG=1 BDEG_DEBUG_LEVELS=1
WALK_SEED=2 timeout 1200 python tools/walk_runs.py w46 > gpurun_out/walk_w46_seed2.log 2>&1; echo "w46 s2 rc $?"; tail -1 gpurun_out/walk_w46_seed2.log | cut -c1-300
timeout 1500 python tools/walk_runs.py w38 > gpurun_out/walk_w38_seed1.log 2>&1; echo "w38 rc $?"; tail -1 gpurun_out/walk_w38_seed1.log | cut -c1-300
timeout 1500 python tools/walk_runs.py w55 > gpurun_out/walk_w55_seed1.log 2>&1; echo "w55 rc $?"; tail -1 gpurun_out/walk_w55_seed1.log | cut -c1-300
