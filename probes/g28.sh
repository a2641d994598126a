for i in 1 2; do timeout 300 python probes/k1t_stage_ms.py 5 >> gpurun_out/g28_stage.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hardening.py -q -x -k "kron_mass or banded or configs or guards" > gpurun_out/g28_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g28_parity.log
