#!/bin/bash
# tests + C4/C3 bench + one full ncu capture of k_lbi (summary + hot SASS): OUT=gpurun_out/<tag>
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/prof}
mkdir -p $OUT
(free -g; nproc; lscpu | grep -i "model name"; df -h /tmp /root 2>/dev/null | tail -3) > $OUT/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest $TESTS -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
fi
for c in ${CONFIGS:-4}; do
  timeout 900 python bench.py --config $c --steps 5 --no-cpu --no-b1 --both 0 ${BENCH_ARGS} > $OUT/bench_c$c.json 2> $OUT/bench_c$c.log
done
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-b1 --both 0 --no-sweep"
for K in ${KERNELS:-k_lbi}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/full_$K -f $CMD > $OUT/ncu_$K.log 2>&1
  python scripts/ncu_summary.py $OUT/full_$K.ncu-rep > $OUT/full_${K}_summary.txt 2>&1
  python scripts/ncu_hot.py $OUT/full_$K.ncu-rep $K 40 > $OUT/full_${K}_hot_sass.txt 2>&1
done
exit 0
