"""TEST INFRASTRUCTURE ONLY (oracle/). Extracts the reference CLI's run_spec
and the helpers it calls (RunSpec, RunResult, matrix_name_of, seeded_rhs,
make_rhs, ms_since — bjgmres_cli.cpp:29-168), unmodified, from where they lie
under /root/reference into oracle/_ref/run_spec_extract.inc (git-ignored,
never committed). tests/cpp/run_spec_dropin_main.cpp compiles that text
against this repo's include/bjgmres/*.hpp: the drop-in check of the C++
solver interface (VERDICT r1 "Next round" 3)."""
import sys

src, dst = sys.argv[1], sys.argv[2]
lines = open(src).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith("struct RunSpec {"))
end = next(i for i, l in enumerate(lines) if l.startswith("json config_json("))
with open(dst, "w") as f:
    f.write(f"// extracted from {src} lines {start + 1}-{end} (unmodified)\n")
    f.write("\n".join(lines[start:end]) + "\n")
