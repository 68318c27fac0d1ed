#!/bin/bash
# f2 on hard queries (C5 sigma = 0.2: nb-ParIS+ vs ParIS+ flat and the index path) and f3 beyond
# HBM (raw in pinned host memory at n = 1.4e8; raw in a file on the local disk): OUT=gpurun_out/<tag>
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=${OUT:-gpurun_out/f3f2}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
(free -g; df -h /tmp) > $OUT/box.txt 2>&1
timeout 900 python bench.py --config 5 --sigma 0.2 --path nb --steps 3 --no-sweep --no-cpu --no-b1 > $OUT/bench_c5_s02_nb.json 2> $OUT/bench_c5_s02_nb.log
timeout 900 python bench.py --config 5 --sigma 0.2 --steps 3 --no-sweep --no-cpu --no-b1 --both 0 > $OUT/bench_c5_s02_index.json 2> $OUT/bench_c5_s02_index.log
for NB in ${NBIG:-120000000 100000000}; do timeout 1500 python bench.py --raw-host --n $NB --steps 3 --no-cpu --no-b1 --both 0 > $OUT/bench_rawhost_big.json 2> $OUT/bench_rawhost_big.log && break; done
(free -g) >> $OUT/box.txt 2>&1
timeout 1500 python bench.py --raw-file /tmp/paris_raw_c4.f32 --n ${NFILE:-60000000} --steps 3 --no-cpu --no-b1 --both 0 > $OUT/bench_rawfile.json 2> $OUT/bench_rawfile.log
rm -f /tmp/paris_raw_c4.f32
exit 0
