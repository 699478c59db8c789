"""Summarise ncu outputs from gpurun_out/ into profiles/ (round-tagged)."""
import csv, io, json, os, subprocess, sys, collections

RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = "profiles"
os.makedirs(OUT, exist_ok=True)

# 1) launch list: per-kernel totals and shares
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
K = hdr.index("Kernel Name"); MN = hdr.index("Metric Name"); MV = hdr.index("Metric Value"); MU = hdr.index("Metric Unit")
tot = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= MV or r[MN] != "gpu__time_duration.sum":
        continue
    name = r[K].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
    v = float(r[MV].replace(",", ""))
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[MU], 1.0)
    tot[name][0] += 1
    tot[name][1] += v * scale
allus = sum(t[1] for t in tot.values())
lines = ["kernel,launches,total_us,mean_us,share"]
for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k},{n},{us:.1f},{us / n:.2f},{us / allus:.3f}")
open(f"{OUT}/{RND}_launch_shares_bench_config1.csv", "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:12]))

# 2) full captures
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]
summary = {}
traffic = {}
for f in sorted(os.listdir("gpurun_out")):
    if not (f.startswith("prof_c") and f.endswith(".ncu-rep")):
        continue
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/{f}", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3:
        continue
    h, u, v = r[0], r[1], r[2]
    d = {}
    for m in want:
        if m in h:
            i = h.index(m)
            d[m] = f"{v[i]} {u[i]}".strip()
    key = f.replace("prof_", "").replace(".ncu-rep", "")
    summary[key] = d
    try:
        rb = float(v[h.index("dram__bytes_read.sum")].replace(",", "")); wb = float(v[h.index("dram__bytes_write.sum")].replace(",", ""))
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rb *= sc.get(u[h.index("dram__bytes_read.sum")], 1); wb *= sc.get(u[h.index("dram__bytes_write.sum")], 1)
        traffic[key] = rb + wb
    except Exception:
        pass
json.dump(summary, open(f"{OUT}/{RND}_ncu_full_summary.json", "w"), indent=1)
print(json.dumps(summary, indent=1)[:3000])
m = {"bj_apply_f32": "c1_k_apply_spk", "spmv_csr_f64": "c1_k_spmv"}
for c in (1, 3):
    t = {nm: traffic.get(f"c{c}_{k.split('_', 1)[1]}") for nm, k in m.items()}
    json.dump(t, open(f"{OUT}/ncu_traffic_config{c}.json", "w"), indent=1)
print(traffic)
