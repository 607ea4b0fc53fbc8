# A/B of the Ozaki-II split: fast (k_split_fast<..., CRT>) vs generic (k_split_sm<8, CX, true>) on C2x30 and C3.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python tests/tools/method_compare.py > gpurun_out/mc_fast.log 2>&1; tail -12 gpurun_out/mc_fast.log
OZAKI_SPLIT=generic timeout 600 python tests/tools/method_compare.py > gpurun_out/mc_generic.log 2>&1; tail -12 gpurun_out/mc_generic.log
