"""A/B of the host region-growing variants (env switches read per call) on
this host: HPBJ_DEBUG phase lines are parsed from stderr of a child per
variant so the timings come from the partitioner itself."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
VARIANTS = [dict(), dict(HPBJ_GROW_PUSHPF="1"), dict(), dict(HPBJ_GROW_PUSHPF="1"), dict(HPBJ_GROW_PF="24")]
for c in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3,2,1").split(",")]:
    for v in VARIANTS:
        env = dict(os.environ, HPBJ_DEBUG="1", **v)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts/gpu/part_debug.py"), str(c)], env=env,
                           capture_output=True, text=True, timeout=600)
        grows = [float(l.split()[2].rstrip(",")) for l in r.stderr.splitlines() if "]   grow " in l]
        tot = [float(l.split()[1]) for l in r.stderr.splitlines() if l.startswith("partition_graph")]
        ell = [l.strip() for l in r.stderr.splitlines() if "ell build" in l][-1:]
        print(f"config {c} {v}: grow ms {grows[1:]} total ms {tot[1:]} {ell}", flush=True)
        if os.environ.get("FULL"):
            print("\n".join(l for l in r.stderr.splitlines()[-12:]), flush=True)
