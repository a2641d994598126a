timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "slab or sharded or peer or k1t" > gpurun_out/g25_slab.log 2>&1; echo "rc=$?" >> gpurun_out/g25_slab.log
timeout 600 python -m pytest tests/test_gpu_hardening.py -q -x > gpurun_out/g25_hard.log 2>&1; echo "rc=$?" >> gpurun_out/g25_hard.log
