#!/bin/bash
# ncu full capture of k_gf inside the C4 bench (variant key 3 = 1)
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/gf}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail -30 $OUT/build.log; exit 1; }
if [ -n "$TESTS" ]; then
timeout ${TEST_TIMEOUT:-600} python -m pytest $TESTS -m gpu -q -x -s > $OUT/pytest_gf.log 2>&1; echo "rc=$?" >> $OUT/pytest_gf.log
grep -a "gf_mma\|candidates:\|passed\|failed\|rc=\|Error\|error" $OUT/pytest_gf.log | tail -25
fi
export PARIS_VARIANT="3=1"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --both 0 --no-sweep --config ${CONFIG:-4}"
timeout 900 ncu --set full --clock-control none --import-source on -k k_gf -s 1 -c 1 -o $OUT/full_k_gf -f $CMD > $OUT/ncu_k_gf.log 2>&1
python scripts/ncu_summary.py $OUT/full_k_gf.ncu-rep > $OUT/full_k_gf_summary.txt 2>&1
python scripts/ncu_hot.py $OUT/full_k_gf.ncu-rep k_gf 60 > $OUT/full_k_gf_hot_sass.txt 2>&1
cat $OUT/full_k_gf_summary.txt
exit 0
