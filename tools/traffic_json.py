"""Fold gpurun_out/traffic/*.csv (ncu launch metrics of the J kernels) into
profiles/ncu_traffic.json: {"<config>_o<order>_<fused|unfused>": bytes per launch}."""
import csv
import glob
import json
import os
import statistics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {"note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant J kernel (median over the "
               "captured launches of that instantiation), ncu --clock-control none on bench.py's own command "
               "(tools/traffic.sh); fused = deposit_current_kernel_v3<..., PM=1|2> (push + detect + J), "
               "unfused = the J-only instantiation (PM=0)"}
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "traffic", "*.csv"))):
    name = os.path.basename(f)[:-4]
    cfg, order = name.rsplit("_o", 1)
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        continue
    h = rows[0]
    k, m, v, u = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    for r in rows[1:]:
        key = (r[h.index("ID")], r[k])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "usecond": 1e3,
                 "msecond": 1e6, "nsecond": 1}.get(r[u], 1)
        per.setdefault(key, {})[r[m]] = float(r[v].replace(",", "")) * scale
    groups = {}
    for (_, kname), d in per.items():
        if "deposit_current_kernel" not in kname:
            continue
        fused = ", 0, " not in kname.split("<", 1)[1]
        groups.setdefault(fused, []).append(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0))
    for fused, vals in groups.items():
        out[f"{cfg}_o{order}_{'fused' if fused else 'unfused'}"] = statistics.median(vals)
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
