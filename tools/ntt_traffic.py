#!/usr/bin/env python
"""DRAM traffic per limb transform of the NTT-family launches (ntt_strided / ntt_contig / ntt_fused /
ntt_ks_inner) of one headline step, from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (bench.py --ncu, one step):
    python tools/ntt_traffic.py launches.csv LIMB_TRANSFORMS_PER_STEP ALG_BYTES_PER_STEP > profiles/ntt_traffic.json
ALG_BYTES_PER_STEP: the bench line's algorithmic NTT bytes per step (transform + fused operands)."""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_launches import kname  # noqa: E402

path, units, alg = sys.argv[1], float(sys.argv[2]), float(sys.argv[3])
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
         "nsecond": 1e-3, "msecond": 1e3}
per, names = collections.defaultdict(dict), {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    names[r[ii]] = kname(r[ki])
byk = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    n = names[i]
    if not n.startswith("ntt_"):
        continue
    b = byk[n.split("<")[0]]
    b[0] += 1
    b[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    b[2] += m.get("gpu__time_duration.sum", 0)
tot = sum(v[1] for v in byk.values())
print(json.dumps({
    "dram_bytes_per_limb_transform": round(tot / units),
    "algorithmic_bytes_per_limb_transform_incl_operands": round(alg / units),
    "traffic_over_algorithmic": tot / alg,
    "per_kernel": {k: {"launches": v[0], "dram_bytes": v[1], "us": v[2]} for k, v in byk.items()},
    "source": "ncu launch list of one headline step (%s): dram__bytes_read.sum + dram__bytes_write.sum of every NTT-family "
              "launch (incl. the fused ModUp pass 2 + key inner product) / %d limb transforms" % (os.path.basename(path), units),
}, indent=1))
