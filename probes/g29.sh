#!/bin/bash
# round-2 re-entry check of HEAD: GPU suite, smoke, stage times, config-5 and config-2 bench lines
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g29_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g29_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g29_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g29_smoke.log
for c in 5 4 3 2; do timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g29_stage.txt 2>&1; done
timeout 600 python bench.py --config 5 --no-cpu-baseline > gpurun_out/g29_bench_c5.json 2> gpurun_out/g29_bench_c5.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/g29_bench_c2.json 2> gpurun_out/g29_bench_c2.err
echo done
