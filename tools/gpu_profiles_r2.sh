# round-2 profile refresh on config0_t10 (bench default): launch list + one full capture of the last Rx run
mkdir -p gpurun_out/prof2
P=gpurun_out/prof2
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $P/gpu.txt
timeout 600 python tools/profile_run.py config0_t10 --warm > $P/plain.log 2>&1; echo "plain rc=$?"; tail -1 $P/plain.log
timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_config0_t10.csv python tools/profile_run.py config0_t10 --warm > /dev/null 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $P/launches_config0_t10.csv > $P/launches_config0_t10_summary.txt; head -30 $P/launches_config0_t10_summary.txt
timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:${KRE:-k_dense_sublayer} --launch-skip ${SKIP:-9} --launch-count 1 -o $P/full_sublayer_config0_t10 python tools/profile_run.py config0_t10 --warm > $P/full.log 2>&1; echo "full rc=$?"
python tools/ncu_summary.py $P/full_sublayer_config0_t10.ncu-rep > $P/full_sublayer_config0_t10_summary.txt; cat $P/full_sublayer_config0_t10_summary.txt
