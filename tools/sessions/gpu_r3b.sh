python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 300 python tools/split_check.py c2 3 > gpurun_out/sc_c2.log 2>&1
timeout 300 python tools/split_check.py c3 3 > gpurun_out/sc_c3.log 2>&1
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --workload c2 --reps 1 > gpurun_out/cyc_c2.log 2>&1
GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 > gpurun_out/c4.log 2>&1
cat gpurun_out/sc_c2.log gpurun_out/sc_c3.log; tail -9 gpurun_out/cyc_c2.log; tail -3 gpurun_out/c4.log
