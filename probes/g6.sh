set -u
mkdir -p gpurun_out
for c in 4 5; do for d in 0 1 2; do FDP_K1T_DIV=$d timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g6_stage.txt 2>&1; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1t or configs or config4 or config5_full_size_oracle" > gpurun_out/g6_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g6_parity.log
echo done
