# SPDX-License-Identifier: Apache-2.0
"""Pretty-print the last JSON line of a bench.py run: headline + per-kernel roofline."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"value {d['value']:.0f} img/s  ms/step {d['ms_per_step']:.3f}  e2e {d['e2e']['value'] if d.get('e2e') else None}  clocks {d['clocks']}")
print("roofline:", {k: v for k, v in d['roofline'].items() if k not in ('algorithmic_per_step',)})
for n, v in sorted(d['kernels'].items(), key=lambda x: -x[1]['ms_per_step']):
    print(f"{n:18s} {v['ms_per_step']:.3f} ms  modmul {v.get('modmul_t_per_s', 0):.2f} T/s  mac {v.get('mac_t_per_s', 0):.2f} T/s"
          f"  hbm {v['hbm_gbs']:.0f} GB/s  frac {v['roofline_frac']:.3f} {v['bound']}")
