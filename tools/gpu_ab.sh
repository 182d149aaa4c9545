# A/B of the per-call device times on C4: abtree/old (previous commit) vs this tree
mkdir -p gpurun_out
(cd abtree/old && SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 8) > gpurun_out/ab_old.txt 2>&1
SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 8 > gpurun_out/ab_new.txt 2>&1
(cd abtree/old && SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 8) > gpurun_out/ab_old2.txt 2>&1
head -30 gpurun_out/ab_old.txt gpurun_out/ab_new.txt gpurun_out/ab_old2.txt
