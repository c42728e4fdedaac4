mkdir -p gpurun_out
PP_DEBUG=1 timeout 600 python tools/profile_run.py config0_t10 --warm 2>&1 | grep -E "dense|branch strings|host wall"
PP_DEBUG=1 timeout 600 python tools/profile_run.py config1 --warm 2>&1 | grep -E "dense|branch strings|host wall"
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_branch_sublayer --launch-skip 9 --launch-count 1 -o gpurun_out/sub_c0t10 python tools/profile_run.py config0_t10 --warm > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
