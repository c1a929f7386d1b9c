# A/B of the dynamic-tail experiment (profiles/r02s4_dyn_tail_experiment.patch must be applied:
# it adds EBS_DYN_ROUNDS; the product build ignores the variable).  Result: profiles/r02s4_dyn_tail_ab.log
for rep in 1 2; do
for r in 0 1 2 3 5 8 100; do
  EBS_DYN_ROUNDS=$r python bench.py --no-cpu --no-extra --steps 100 --warmup 5 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('dyn_rounds=$r value %.2f GDoF/s  step %.1f us  sell %.1f us  gather %.1f us  exact %.2f  e2e %.2f' % (d['value'], d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['roofline']['gather_kernel_ms']*1e3, d['exact_mode']['value'], d['e2e']['value']))
"
done; done
