# A/B of two library builds (variants/v_old, variants/v_new) on the default C4
# bench: step time and the per-kernel eager profile of the listed kernels
for v in ${VARS:-v_old v_new v_old v_new}; do
MLBM_LIB=variants/$v/libmlbm_b200.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read());k=d['kernels']
print('$v', d['ms_per_step'], d['graph']['step_ms']['median'], ' '.join('%s=%.3f'%(n,k[n]['ms_per_step']) for n in ('${KERNELS:-g2p p2g}'.split()) if n in k))"
done
