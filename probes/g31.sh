#!/bin/bash
set -u
mkdir -p gpurun_out /tmp/ncu
timeout 300 python probes/k1t_stage_ms.py 5 >> gpurun_out/g31_stage.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mass_tile -c 2 -o /tmp/ncu/k3t -f python probes/k1t_stage_ms.py 5 > gpurun_out/g31_ncu.log 2>&1
ncu -i /tmp/ncu/k3t.ncu-rep --page details --csv > gpurun_out/g31_k3t_details.csv 2>&1
ncu -i /tmp/ncu/k3t.ncu-rep --page raw --csv > gpurun_out/g31_k3t_raw.csv 2>&1
ncu -i /tmp/ncu/k3t.ncu-rep --page source --csv --print-source sass > gpurun_out/g31_k3t_src.csv 2>&1
echo done
