python -c "import __graft_entry__ as g; g.build()" || exit 1
RND=r02 bash scripts/profile_round.sh > gpurun_out/r02_profile_round.log 2>&1
