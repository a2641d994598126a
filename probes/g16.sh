for c in 5 3; do timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g16_stage.txt 2>&1; done
for c in 5; do FDP_MASS_FIBER=1 timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g16_stage.txt 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "kron_mass or configs or config5_full_size or slab or k1_sized_pressure" > gpurun_out/g16_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g16_parity.log
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_gmres.py -q -x > gpurun_out/g16_krylov.log 2>&1; echo "rc=$?" >> gpurun_out/g16_krylov.log
