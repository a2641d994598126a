timeout 1200 python -m pytest tests/test_gpu_hardening.py -q -x > gpurun_out/g19_hardening.log 2>&1; echo "rc=$?" >> gpurun_out/g19_hardening.log
