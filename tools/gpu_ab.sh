# A/B of per-call device times on C4: abtree/prev (last commit) vs this tree, interleaved
mkdir -p gpurun_out
for i in 1 2; do
(cd abtree/prev && SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 8) > gpurun_out/ab_prev_$i.txt 2>&1
SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 8 > gpurun_out/ab_new_$i.txt 2>&1
done
head -8 gpurun_out/ab_prev_*.txt gpurun_out/ab_new_*.txt
