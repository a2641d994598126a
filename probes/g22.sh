for c in 5; do timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g22_stage.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kron_mass or configs" > gpurun_out/g22_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g22_parity.log
