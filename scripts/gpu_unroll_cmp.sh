cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for C in C2 C5 C4; do for U in 1 2 4; do
NLSP_UNROLL=$U timeout 300 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/u_${C}_$U.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/u_${C}_$U.json')); print('$C', 'unroll=$U', d['value'], d['iterations_per_solve'], d['gpu_launches'], d['clocks']['sm_mhz'])"
done; done
