#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
OUT=gpurun_out/r2l
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_index.py -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
B="python bench.py --steps 5 --no-cpu --no-b1 --both 0"
timeout 600 $B --paa 64 --no-raw16 > $OUT/c4_paa64.json 2> $OUT/c4_paa64.log
timeout 600 $B --paa 32 --no-raw16 > $OUT/c4_paa32.json 2> $OUT/c4_paa32.log
timeout 600 $B --paa 64 > $OUT/c4_paa64_bf16.json 2> $OUT/c4_paa64_bf16.log
timeout 600 $B --config 3 --paa 32 --no-raw16 > $OUT/c3_paa32.json 2> $OUT/c3_paa32.log
timeout 600 $B --config 3 --paa 64 --no-raw16 > $OUT/c3_paa64.json 2> $OUT/c3_paa64.log
timeout 600 $B --config 5 --paa 64 --no-raw16 --no-sweep > $OUT/c5_paa64.json 2> $OUT/c5_paa64.log
timeout 600 $B --config 2 --paa 64 --no-raw16 --no-sweep > $OUT/c2_paa64.json 2> $OUT/c2_paa64.log
exit 0
