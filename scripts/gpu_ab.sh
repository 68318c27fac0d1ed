#!/bin/bash
# A/B of a build flag: tests + C4 benches with the default build, then with ABFLAG (e.g. "PARIS_REFQ_CTAS=4")
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2009_00166_b200.build --force > gpurun_out/build_a.log 2>&1
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_a.log
for c in ${CONFIGS:-4}; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-b1 > gpurun_out/ab_a_c$c.json 2> gpurun_out/ab_a_c$c.log
done
env $ABFLAG python -m paper_2009_00166_b200.build --force > gpurun_out/build_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log
for c in ${CONFIGS:-4}; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-b1 > gpurun_out/ab_b_c$c.json 2> gpurun_out/ab_b_c$c.log
done
python -m paper_2009_00166_b200.build --force > gpurun_out/build_restore.log 2>&1  # leave the default build behind
exit 0
