set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "slab or sharded or peer" > gpurun_out/g3_slab.log 2>&1; echo "rc=$?" >> gpurun_out/g3_slab.log
timeout 300 python probes/sanitize_cases.py slab > gpurun_out/g3_sancases.log 2>&1; echo "rc=$?" >> gpurun_out/g3_sancases.log
