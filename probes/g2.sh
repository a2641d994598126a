set -u
mkdir -p gpurun_out
./probes/tma_odd > gpurun_out/g2_tma_odd.txt 2>&1; echo "tma_odd rc=$?" >> gpurun_out/g2_tma_odd.txt
for c in 4 5; do for d in 0 1 2; do
FDP_K1T_DBG=$d timeout 300 python probes/k1t_stage_ms.py $c >> gpurun_out/g2_stage.txt 2>&1
done; done
echo done
