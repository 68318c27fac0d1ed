#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python scripts/prof_lb.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_lbt|k_summarize|k_refine" -c 6 -o gpurun_out/prof_lb -f python scripts/prof_lb.py > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof_ncu.log
