timeout 900 python bench.py --no-other-configs --no-cpu-baseline --steps 5 > gpurun_out/bench_q.out 2> gpurun_out/bench_q.err
tail -1 gpurun_out/bench_q.out | python3 -c "
import json,sys; d=json.loads(sys.stdin.read())
o=d.get('offload',{})
for k in ('config4_lora_step','config5_blockwise'):
    v=o.get(k,{}); print(k, {x:v.get(x) for x in ('step_s','frac_of_duplex_bound','plan_copy_bound_s','frac_of_plan_copy_bound','dependency_bound_s','frac_of_dependency_bound')})
print('value', d.get('value'))
"
tail -3 gpurun_out/bench_q.err
