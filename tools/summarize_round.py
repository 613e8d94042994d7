"""Summarise a round's evidence directory (tools/jobs output copied under profiles/) into
profiles/<dir>/summary.json and print the DESIGN.md §5 tables. Usage:
  python tools/summarize_round.py profiles/r2/final"""
import csv
import json
import os
import sys

D = sys.argv[1]


def line(name):
    p = os.path.join(D, name + ".json")
    if not os.path.exists(p):
        return None
    rows = [x for x in open(p).read().splitlines() if x.strip().startswith("{")]
    return json.loads(rows[-1]) if rows else None


out = {}
print("| config | N | µs/step (K=20, driver run) | K=200 | K=2000 | HBM frac at K=20 / K=2000 | aug samples/s (K=20) | e2e aug/s | update µs/step |")
print("|---|---|---|---|---|---|---|---|---|")
for name in ["bench_n1", "bench_n2", "bench_n4", "bench_config_c1", "bench_config_c3", "bench_config_c4r7",
             "bench_config_c4r14", "bench_config_c4", "bench_config_c5"]:
    d = line(name)
    if not d:
        continue
    sw = {x["steps"]: x["us_per_step"] for x in d.get("steps_sweep", [])}
    rf = d["roofline"]
    bps = rf["algorithmic_bytes_per_step"]
    us = d["ms_per_step"] * 1000
    f2000 = bps / (sw[2000] * 1e-6) / 1e9 / rf["peak"] if 2000 in sw else None
    cfg = d["config"]["workload"]
    out[name] = {"us_per_step": us, "sweep": sw, "frac": rf["frac"], "frac_2000": f2000, "value": d["value"],
                 "e2e": d["e2e"]["value"], "update_us_per_step": d.get("update_us_per_step"),
                 "clocks": d.get("clocks"), "workload": cfg, "n_gpus": d["n_gpus"]}
    print(f"| {cfg} | {d['n_gpus']} | {us:.2f} | {sw.get(200, float('nan')):.2f} | {sw.get(2000, float('nan')):.2f} | "
          f"{rf['frac']:.2f} / {f2000 if f2000 is None else round(f2000, 2)} | {d['value'] / 1e6:.2f} M | "
          f"{d['e2e']['value'] / 1e3:.0f} K | {d.get('update_us_per_step') if d.get('update_us_per_step') is None else round(d['update_us_per_step'], 2)} |")
print()
for name in ["bench_ref_n1", "bench_ref_n2", "bench_ref_n4"]:
    d = line(name)
    if d:
        cb = d["cpu_baseline"]
        out[name] = {"value": d["value"], "cores": cb.get("cores"), "n_workers": cb.get("n_workers"),
                     "cpu": cb.get("cpu_model"), "nproc": cb.get("nproc")}
        print(f"reference arm N={d['n_gpus']}: {d['value'] / 1e3:.1f} K aug/s ({cb.get('cores')} threads, "
              f"{cb.get('cpu_model')}, nproc {cb.get('nproc')})")
d = line("bench_n1")
if d and d.get("update", {}).get("cpp_facade"):
    out["update_cpp"] = d["update"]["cpp_facade"]
    print("update (C++ facade):", json.dumps(d["update"]["cpp_facade"]))
raw = os.path.join(D, "ncu_run_r2final_raw.csv")
if os.path.exists(raw):
    rows = list(csv.reader(open(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {}
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active"):
        if k in h:
            m[k] = (v[h.index(k)], u[h.index(k)])
    out["ncu_full_capture_200_steps"] = m
    print("ncu full capture (200-step instance):", m)
json.dump(out, open(os.path.join(D, "summary.json"), "w"), indent=1)
