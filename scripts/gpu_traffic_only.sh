#!/bin/bash
# Re-capture the DRAM traffic JSON (ncu --set full of the roofline kernels) for the current build, after
# a quick check: the filter's tests, a parity subset, smoke, and two default bench lines.
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/ev7}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
sha256sum paper_2009_00166_b200/libparis.so > $OUT/lib_sha.txt
timeout 900 python -m pytest tests/test_gpu_gf.py tests/test_gpu_parity.py tests/test_gpu_index.py tests/test_abi.py -m gpu -q > $OUT/pytest_subset.log 2>&1; echo "rc=$?" >> $OUT/pytest_subset.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default_pre.json 2> $OUT/bench_default_pre.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-b1 --both 0 --no-sweep"
CMDF="python bench.py --steps 2 --warmup 3 --no-cpu --both 0 --no-sweep --path flat"
for spec in "k_lbi 1 1" "k_refine1m 2 2" "k_summarize_seg 1 1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -o $OUT/full_c4_$1 -f $CMD > $OUT/ncu_full_$1.log 2>&1
  python scripts/ncu_summary.py $OUT/full_c4_$1.ncu-rep > $OUT/full_c4_$1_summary.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k k_gf -s 1 -c 1 -o $OUT/full_c4_k_gf -f $CMDF > $OUT/ncu_full_k_gf.log 2>&1
python scripts/ncu_summary.py $OUT/full_c4_k_gf.ncu-rep > $OUT/full_c4_k_gf_summary.txt 2>&1
python scripts/ncu_hot.py $OUT/full_c4_k_gf.ncu-rep k_gf 40 > $OUT/full_c4_k_gf_hot_sass.txt 2>&1
python scripts/ncu_traffic.py $OUT > $OUT/ncu_traffic.json 2> $OUT/ncu_traffic.log && cp $OUT/ncu_traffic.json profiles/ncu_traffic.json
rm -f $OUT/*.ncu-rep
sleep 20
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.log
python scripts/bench_brief.py $OUT/bench_*.json > $OUT/brief.txt 2>&1
exit 0
