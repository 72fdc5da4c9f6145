# round evidence: GPU tests, smoke, default bench line, reference arm, ncu launch list + captures; tag $1
T=${1:-r14}
set -x
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputest_$T.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/gputest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/bench_$T.log 2> gpurun_out/bench_$T.err; echo bench rc $?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$T.log 2>&1; echo ref rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 1 --no-sub --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu launches rc $?
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/prof_$T -f python tools/profile_workload.py c2 > gpurun_out/ncu_c2_$T.log 2>&1; echo ncu c2 rc $?
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
timeout 600 ncu --profile-from-start off $M -o gpurun_out/attack_$T -f python tools/profile_workload.py attack > gpurun_out/ncu_attack_$T.log 2>&1; echo ncu attack rc $?
timeout 900 python bench.py --workload c3 > gpurun_out/bench_c3_$T.log 2> gpurun_out/bench_c3_$T.err; echo c3 rc $?
timeout 1200 python bench.py --workload c5 --steps 5 --warmup 1 > gpurun_out/bench_c5_$T.log 2> gpurun_out/bench_c5_$T.err; echo c5 rc $?
