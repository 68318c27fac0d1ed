#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_index.py -q -x > gpurun_out/pytest_idx.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_idx.log
CMD="python bench.py --config 4 --steps 2 --warmup 3 --path index --no-cpu --no-b1 --both 0 $EXTRA"
$CMD > gpurun_out/pidx_plain.json 2> gpurun_out/pidx_plain.log && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_lbi} -s ${KSKIP:-1} -c ${KCOUNT:-1} -o gpurun_out/full_c4_idx -f $CMD > gpurun_out/pidx_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/pidx_ncu.log
exit 0
