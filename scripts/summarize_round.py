"""Summarise a round's ncu outputs (scripts/profile_round.sh) into profiles/:
launch shares of the bench step, per-kernel full-capture metrics, the DRAM
traffic per launch used by bench.py's roofline, and SASS listings."""
import collections, csv, io, json, os, re, subprocess, sys

RND = sys.argv[1] if len(sys.argv) > 1 else "r01"
SRC = os.environ.get("SRC", "gpurun_out")
OUT = os.environ.get("OUT", "profiles")
os.makedirs(OUT, exist_ok=True)
SC = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    n = name.split("(")[0].replace("void ", "").replace("hpbj::", "").replace("unnamed>::", "")
    return re.sub(r"spk::", "", n)


# 1) launch shares of the bench (BENCH_CONFIG, default 3; NOGRAPH) -------------------------
p = f"{SRC}/{RND}_launches_bench.csv"
if os.path.exists(p):
    rows = [r for r in csv.reader(open(p)) if len(r) > 10]
    h = rows[0]
    K, MU, MV = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        tot[short(r[K]).lstrip("<")][0] += 1
        tot[short(r[K]).lstrip("<")][1] += float(r[MV].replace(",", "")) * SC.get(r[MU], 1.0)
    allus = sum(t[1] for t in tot.values())
    lines = ["kernel,launches,total_us,mean_us,share"]
    for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"\"{k}\",{n},{us:.1f},{us / n:.2f},{us / allus:.4f}")
    open(f"{OUT}/{RND}_launch_shares_bench_config{os.environ.get('BENCH_CONFIG', '3')}.csv", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:14]))

# 2) full captures -----------------------------------------------------------
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
BS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
summary, traffic = {}, collections.defaultdict(dict)
kmap = {"apply": "bj_apply_f32", "spmv": "spmv_csr_f64", "icwy": "arnoldi_mgs_f64", "mgs": "arnoldi_mgs_f64",
        "lu": "block_lu_f32", "spk_build": "spk_build",
        "arnoldi_cycle": "arnoldi_cycle_fused"}
for f in sorted(os.listdir(SRC)):
    if not (f.startswith(f"{RND}_prof_") and f.endswith(".ncu-rep")):
        continue
    key = f[len(f"{RND}_prof_"):-len(".ncu-rep")]
    raw = subprocess.run(["ncu", "-i", f"{SRC}/{f}", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3:
        continue
    h, u, v = r[0], r[1], r[2]
    d = {"kernel": short(v[h.index("Kernel Name")])}
    for m in want:
        if m in h:
            i = h.index(m)
            d[m] = f"{v[i]} {u[i]}".strip()
    try:
        rb = float(v[h.index("dram__bytes_read.sum")].replace(",", "")) * BS.get(u[h.index("dram__bytes_read.sum")], 1)
        wb = float(v[h.index("dram__bytes_write.sum")].replace(",", "")) * BS.get(u[h.index("dram__bytes_write.sum")], 1)
        d["dram_bytes"] = rb + wb
        cfg, kind = key.split("_", 1)
        if kind in kmap:
            traffic[cfg][kmap[kind]] = rb + wb
    except Exception as e:
        print("traffic parse failed", key, e)
    summary[key] = d
json.dump(summary, open(f"{OUT}/{RND}_ncu_full_summary.json", "w"), indent=1)
for cfg, t in traffic.items():
    c = cfg[1:]
    path = f"{OUT}/ncu_traffic_config{c}.json"
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(t)
    if "arnoldi_cycle_fused" in t:  # the capture is the first launch: one full cycle of m steps (config 1: m = 50)
        old.setdefault("arnoldi_cycle_fused_steps", 50)
    old["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full ({RND}); "
                    "arnoldi_cycle_fused: one launch = one restart cycle (the first, m steps)")
    json.dump(old, open(path, "w"), indent=1)
for k, d in summary.items():
    print(k, d.get("kernel"), d.get("gpu__time_duration.sum"), "dram", d.get("dram_bytes"))

# 3) SASS listings of the shipped kernels -----------------------------------
so = "paper_2509_09139_b200/lib/libhpbj.so"
if os.path.exists(so):
    os.makedirs(f"{OUT}/sass_{RND}", exist_ok=True)
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    index = []
    hot = ("k_apply_spk<float, unsigned short, false, false, SrcDown", "k_apply_spk<float, unsigned short, false, true, SrcDown",
           "k_apply_spk<float, unsigned short, true, false, SrcDown", "k_arnoldi_cycle<false", "k_spmv<1, float", "k_spmv<2, float",
           "k_icwy<true", "k_mgs<true", "k_block_lu_ll", "k_block_lu_pair<3", "k_spk_build<true, unsigned short",
           "k_spk_build<false")
    for fn in funcs[1:]:
        name = fn.split("\n", 1)[0].strip()
        dn = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        tag = short(dn)
        base = re.sub(r"[^A-Za-z0-9_]+", "_", tag)[:80]
        nins = len(re.findall(r"/\*[0-9a-f]{4,}\*/", fn))
        index.append((tag, nins, base if tag.startswith(hot) else None))
        if not tag.startswith(hot):
            continue
        body = []
        for line in fn.split("\n"):
            line = re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", line).rstrip()
            if line.strip():
                body.append(line)
        open(f"{OUT}/sass_{RND}/{base}.sass", "w").write(f"// {dn}\n" + "\n".join(body) + "\n")
    with open(f"{OUT}/sass_{RND}/INDEX.md", "w") as f:
        f.write(f"# SASS listings ({RND}), `cuobjdump -sass {so}`\n\n| kernel | instructions | file |\n|---|---|---|\n")
        for tag, nins, base in sorted(index):
            f.write(f"| `{tag}` | {nins} | {base + '.sass' if base else '(not kept)'} |\n")
    print(len(index), "SASS listings")
