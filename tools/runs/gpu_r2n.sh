#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not twins" > gpurun_out/r2n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_tests.log
tail -2 gpurun_out/r2n_tests.log
bash tools/ab_bench.sh adaptive scratch/libbdeg_cur.so -
BDEG_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2n_bench_share2.json 2> gpurun_out/r2n_bench_share2.err; echo "share2 rc=$?"; tail -c 700 gpurun_out/r2n_bench_share2.json; tail -3 gpurun_out/r2n_bench_share2.err
