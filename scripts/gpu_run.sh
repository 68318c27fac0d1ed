#!/bin/bash
# generic GPU pass: build, gpu tests, smoke, benches (args: list of configs)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
for c in $CONFIGS; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 $BENCH_ARGS > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.log
done
exit 0
