#!/bin/bash
# iteration pass: quick GPU tests, then C4/C5 benches (+ an A/B arg on C4)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -m paper_2009_00166_b200.build --force > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py ${TESTS:-} > gpurun_out/pytest_iter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_iter.log
for c in ${CONFIGS:-4 5}; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-b1 > gpurun_out/it_c$c.json 2> gpurun_out/it_c$c.log
done
if [ -n "$AB" ]; then
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-b1 $AB > gpurun_out/it_ab_c4.json 2> gpurun_out/it_ab_c4.log
fi
exit 0
