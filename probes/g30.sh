#!/bin/bash
# K3t (tile) check: its tests, the banded paths of the parity suite, config-5 stage times with and without it
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_k3.py -q -x > gpurun_out/g30_k3.log 2>&1; echo "rc=$?" >> gpurun_out/g30_k3.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py -q -x -k "kron_mass or banded or configs or guards or slab" > gpurun_out/g30_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g30_parity.log
for i in 1 2; do timeout 300 python probes/k1t_stage_ms.py 5 >> gpurun_out/g30_stage.txt 2>&1; done
FDP_K3_SWEEP=1 timeout 300 python probes/k1t_stage_ms.py 5 >> gpurun_out/g30_stage.txt 2>&1
echo done
