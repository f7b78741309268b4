"""Runs on the GPU box: DRAM traffic per launch of the flux kernels at every
point bench.py's order / precision sweep visits, from ncu
(dram__bytes_read.sum + dram__bytes_write.sum, --clock-control none). Writes
gpurun_out/traffic.json with the keys bench.py looks up
(kernel/N<order>/<precision>/<case>); copy it to profiles/traffic.json."""
import csv
import io
import json
import subprocess
import sys

points = [(o, p, "bubble", "stage") for o in (2, 3, 4, 5, 6, 7) for p in ("f64", "f32")]
points += [(4, "f64", "bubble", "split"), (4, "f32", "bubble", "split"), (4, "f64", "bubble", "fused"),
           (4, "f64", "baroclinic", "stage")]
table = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over the launches of one LSRK "
                  "step), ncu --clock-control none, tools/collect_traffic.py; meshes: SURVEY.md 8(d) config 2"}
for order, prec, case, path in points:
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control", "none",
           "-k", "regex:rhs_kernel|axpy_kernel", "--csv", "python", "tools/traffic_probe.py", str(order), prec, case, path]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900).stdout
    rows = list(csv.reader(io.StringIO(out[out.find('"ID"'):])))
    if not rows:
        print("no rows for", order, prec, case, path, file=sys.stderr)
        continue
    idx = {h: i for i, h in enumerate(rows[0])}
    per = {}
    for r in rows[1:]:
        if len(r) < len(rows[0]):
            continue
        name, val, unit = r[idx["Kernel Name"]], float(r[idx["Metric Value"]].replace(",", "")), r[idx["Metric Unit"]]
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        kid = r[idx["ID"]]
        per.setdefault((kid, name), 0.0)
        per[(kid, name)] += val * scale
    groups = {}
    for (kid, name), b in per.items():
        if "axpy" in name:
            key = "update"
        else:
            args = name[name.find("<") + 1:name.rfind(">")].replace("(bool)", "").replace("(int)", "").split(",")
            # rhs_kernel<Real, NQ, EPB, MINB, VOL, SURF, RUNG>
            vol, surf = args[4].strip() in ("1", "true"), args[5].strip() in ("1", "true")
            key = path if (vol and surf) else ("volume" if vol else "surface")
        groups.setdefault(key, []).append(b)
    for key, vals in groups.items():
        table[f"{key}/N{order}/{prec}/{case}"] = sum(vals) / len(vals)
        print(f"{key}/N{order}/{prec}/{case}: {sum(vals) / len(vals) / 1e9:.3f} GB over {len(vals)} launches", flush=True)
    with open("gpurun_out/traffic.json", "w") as f:
        json.dump(table, f, indent=1)
