mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_branch_sublayer --launch-skip 4 --launch-count 1 -o gpurun_out/sub_last2 python tools/profile_run.py config1 --warm > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
