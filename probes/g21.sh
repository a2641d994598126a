for c in 5 4; do FDP_LIB_PATH=paper_1712_00403_b200/libfdp_prof.so timeout 300 python probes/k1t_roles.py $c >> gpurun_out/g21_roles.txt 2>&1; done
for c in 5 4; do timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g21_stage.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1t or configs or config4 or config5_full_size_oracle or slab" > gpurun_out/g21_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g21_parity.log
