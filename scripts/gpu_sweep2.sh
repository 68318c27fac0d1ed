#!/bin/bash
# build-flag sweep with GPU index tests on the first variant: VARIANTS="A=1,B=2 ..."
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
i=0
for v in $VARIANTS; do
  i=$((i+1))
  env $(echo $v | tr ',' ' ') python -m paper_2009_00166_b200.build --force > gpurun_out/sw_build_$i.log 2>&1
  if [ $i -eq 1 ]; then timeout 900 python -m pytest tests/test_gpu_index.py -q -x > gpurun_out/sw_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sw_pytest.log; fi
  echo "$v" > gpurun_out/sw_$i.txt
  timeout 900 python bench.py --config ${CONFIG:-4} --steps 5 --warmup 3 --no-cpu --no-b1 --both 0 $BARGS >> gpurun_out/sw_$i.txt 2> gpurun_out/sw_$i.log
done
exit 0
