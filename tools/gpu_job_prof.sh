# one full ncu capture of the C2 bank step (every kernel), tag from $1
T=${1:-r14}
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/prof_$T -f python tools/profile_workload.py c2 > gpurun_out/ncu_c2_$T.log 2>&1; echo ncu c2 rc $?
tail -2 gpurun_out/ncu_c2_$T.log
