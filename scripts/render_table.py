"""Render profiles/<round>_per_config.json (bench.py --report-all) as a markdown table."""
import json
import sys

d = json.load(open(sys.argv[1]))
peak = d["peak_gbs"]
print(f"HBM peak (MEASURED_PEAKS.json): {peak:.0f} GB/s; reference CPU: {d['cores']} host cores.\n")
print("| cfg | n | its | partition (host) ms | setup (device) ms | solve ms | us/iter | ms/system | "
      "apply GB/s (frac) | SpMV GB/s (frac) | MGS GB/s | fused cycle GB/s (frac) | reference CPU ms/system |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for c, r in d["configs"].items():
    b = r["breakdown_ms"]
    k = r["kernels"]

    def g(name):
        x = k.get(name)
        if not x or x.get("gbs") is None:
            return "—"
        return f"{x['gbs']:.0f} ({x['hbm_frac']:.2f})"

    mg = k.get("arnoldi_mgs_f64", {}).get("gbs")
    cpu = r.get("cpu_reference")
    cpus = "—"
    if cpu:
        cpus = f"{cpu['ms_per_system']:.0f}" + ("" if cpu["partition"].startswith("reference") else " (partition skipped†)")
    print(f"| {c} | {r['n']:,} | {r['iterations']} | {b['partition_host']:.1f} | {b['bj_setup']:.1f} | "
          f"{b['solve']:.1f} | {b['per_iteration_us']:.0f} | {r['ms_per_system']:.1f} | {g('bj_apply_f32')} | "
          f"{g('spmv_csr_f64')} | {mg:.0f} | {g('arnoldi_cycle_fused')} | {cpus} |" if mg else
          f"| {c} | {r['n']:,} | {r['iterations']} | {b['partition_host']:.1f} | {b['bj_setup']:.1f} | "
          f"{b['solve']:.1f} | {b['per_iteration_us']:.0f} | {r['ms_per_system']:.1f} | {g('bj_apply_f32')} | "
          f"{g('spmv_csr_f64')} | — | {g('arnoldi_cycle_fused')} | {cpus} |")
    if "sequence" in r:
        q = r["sequence"]
        print(f"| 4 (64-step sequence) | | {min(q['iterations'])}-{max(q['iterations'])} | (once) | refactor | | | "
              f"{q['per_step_ms_mean']:.2f}/step, {q['total_ms']:.0f} total | | | | | |")
