#!/bin/bash
# Tensor-core filter (k_gf) iteration: its tests, then C4 bench lines with and without it.
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/gf}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail -30 $OUT/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-600} python -m pytest ${TESTS:-tests/test_gpu_gf.py} -m gpu -q -x -s > $OUT/pytest_gf.log 2>&1; echo "rc=$?" >> $OUT/pytest_gf.log
grep -a "gf_mma\|candidates:\|passed\|failed\|rc=\|Error\|error" $OUT/pytest_gf.log | tail -25
if [ -n "$BENCH" ]; then
  for c in ${CONFIGS:-4}; do
    timeout 900 python bench.py --config $c --steps ${STEPS:-10} --no-cpu ${BENCH_ARGS} > $OUT/bench_c$c.json 2> $OUT/bench_c$c.log
    PARIS_VARIANT="3=1" timeout 900 python bench.py --config $c --steps ${STEPS:-10} --no-cpu ${BENCH_ARGS} > $OUT/bench_c${c}_gf.json 2> $OUT/bench_c${c}_gf.log
  done
  python scripts/bench_brief.py $OUT/*.json 2>&1 | tee $OUT/brief.txt
fi
exit 0
