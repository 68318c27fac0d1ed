#!/bin/bash
# One build -> measure iteration: build, selected GPU tests, C4 bench lines (+ optional A/B env),
# optional ncu full captures of named kernels.  OUT=gpurun_out/<tag> TESTS="tests/x.py ..."
# AB="PARIS_X=1" KERNELS="k_lbi k_lb1t" CONFIGS="4 3"
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/iter}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail -30 $OUT/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest $TESTS -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
for c in ${CONFIGS:-4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --no-cpu ${BENCH_ARGS} > $OUT/bench_c$c.json 2> $OUT/bench_c$c.log
  if [ -n "$AB" ]; then
    env $AB timeout 900 python bench.py --config $c --steps ${STEPS:-10} --no-cpu ${BENCH_ARGS} > $OUT/bench_c${c}_ab.json 2> $OUT/bench_c${c}_ab.log
  fi
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --both 0 --no-sweep ${NCU_ARGS}"
for K in ${KERNELS}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/full_$K -f $CMD > $OUT/ncu_$K.log 2>&1
  python scripts/ncu_summary.py $OUT/full_$K.ncu-rep > $OUT/full_${K}_summary.txt 2>&1
  python scripts/ncu_hot.py $OUT/full_$K.ncu-rep $K 40 > $OUT/full_${K}_hot_sass.txt 2>&1
done
python scripts/bench_brief.py $OUT/*.json 2>&1 | tee $OUT/brief.txt
exit 0
