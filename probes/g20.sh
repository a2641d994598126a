for c in 5 4; do FDP_LIB_PATH=paper_1712_00403_b200/libfdp_prof.so timeout 300 python probes/k1t_roles.py $c >> gpurun_out/g20_roles.txt 2>&1; done
