#!/bin/bash
# final check: build as the driver does, all GPU tests, smoke, the default bench line
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/fin
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin/smoke.log
timeout 900 python bench.py > gpurun_out/fin/bench_default.json 2> gpurun_out/fin/bench_default.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/fin/bench_torchrun1.json 2> gpurun_out/fin/bench_torchrun1.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin/bench_reference.json 2> gpurun_out/fin/bench_reference.log
exit 0
