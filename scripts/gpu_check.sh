#!/bin/bash
# build + smoke + selected GPU tests + default bench (+ extra bench configs): OUT=gpurun_out/<tag>
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/chk}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-2400} python -m pytest $TESTS -m gpu -q -x ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
fi
for c in ${CONFIGS:-4}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS} > $OUT/bench_c$c.json 2> $OUT/bench_c$c.log
done
exit 0
