#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_index.py -q -x > gpurun_out/pytest_idx.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_idx.log
for c in ${CONFIGS:-4}; do
for v in ${VARIANTS:-"0 4096" "1 4096"}; do
  set -- $v
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --path index --no-cpu --no-b1 --index-seeds $2 > gpurun_out/tune_c${c}_g$1_s$2.json 2> gpurun_out/tune_c${c}_g$1_s$2.log
done
done
exit 0
