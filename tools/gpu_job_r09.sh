set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gputest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/gputest.log
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/prof_r09 -f python tools/profile_workload.py c2 > gpurun_out/ncu_c2.log 2>&1; echo ncu c2 rc $?
timeout 900 ncu --profile-from-start off $M --replay-mode application -o gpurun_out/c4_r09 -f python tools/profile_workload.py c4 > gpurun_out/ncu_c4.log 2>&1; echo ncu c4 rc $?
timeout 600 ncu --profile-from-start off $M -o gpurun_out/attack_r09 -f python tools/profile_workload.py attack > gpurun_out/ncu_attack.log 2>&1; echo ncu attack rc $?
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/attack_full_r09 -f python tools/profile_workload.py attack > gpurun_out/ncu_attack_full.log 2>&1; echo ncu attackfull rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r09.csv python bench.py --steps 2 --warmup 1 --no-sub --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu launches rc $?
