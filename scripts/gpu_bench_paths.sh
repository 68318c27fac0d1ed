#!/bin/bash
# benches of both query paths for $CONFIGS
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in $CONFIGS; do
  for pth in ${PATHS:-flat index}; do
    timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --path $pth $BENCH_ARGS > gpurun_out/bench_c${c}_$pth.json 2> gpurun_out/bench_c${c}_$pth.log
  done
done
exit 0
