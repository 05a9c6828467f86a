# A/B of scratch libraries on the C5 / W26 bench (ms per step)
cd $GRAFT_REPO_ROOT
ms() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f' % d['ms_per_step'])"; }
for i in 1 2 3; do
  for lib in paper_1501_02237_b200/libbdeg.so ${LIBS}; do
    echo "$lib c5 $(BDEG_LIB=$lib python bench.py --no-cpu-baseline 2>&1 | ms) w26 $(BDEG_LIB=$lib python bench.py --workload w26 --steps 3 --no-cpu-baseline 2>&1 | ms)"
  done
done
