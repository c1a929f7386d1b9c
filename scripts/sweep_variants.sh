#!/bin/bash
# Time the bench (C2 residual + C3/C4/C5 solvers) for each prebuilt libebs variant.
mkdir -p gpurun_out
for f in paper_1911_03973_b200/variants/libebs_*.so paper_1911_03973_b200/libebs.so; do
  n=$(basename $f .so)
  EBS_LIB_PATH=$PWD/$f timeout 300 python bench.py --steps 100 --no-cpu --extra > gpurun_out/sweep_$n.json 2> gpurun_out/sweep_$n.err
  python - "$n" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweep_{n}.json").read().strip().splitlines()[-1])
    s = d.get("solvers", {})
    print(n, "C2 %.2f GDoF/s kern %.1f us frac %.3f exact %.2f" % (d["value"], d["roofline"]["kernel_ms"]*1e3, d["roofline"]["frac"], d["exact_mode"]["value"]),
          " | ".join(f"{k}: {v.get('it_per_s',0):.0f} it/s {v.get('frac_of_peak',0):.3f}" for k, v in s.items()))
except Exception as e:
    print(n, "FAILED", e)
PY
done
