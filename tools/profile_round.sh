#!/bin/bash
# Round measurement recipe (run under gpurun on one B200):
#   tools/profile_round.sh r02
# 1. the contract bench line, 2. the plain run of the profiled command,
# 3. the ncu launch list of that command, 4. one ncu --set full capture of the
# SL kernel (+ fp64 / local-memory instruction counters), 5. per-kernel DRAM
# bytes and durations of the loop body. Outputs land in gpurun_out/;
# summaries are made locally with tools/ncu_summary.py / tools/loop_roofline.py
# and committed under profiles/.
R=${1:-r02}
python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-loop"
$CMD > gpurun_out/plain_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sl_step_|resync_kernel|zt_|FillFunctor" \
    -c 60 --csv --log-file gpurun_out/launches_$R.csv $CMD > gpurun_out/ncu_launch_$R.log 2>&1
ncu --set full --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum \
    --clock-control none --import-source on -k regex:sl_step_zt -s 3 -c 1 \
    -o gpurun_out/sl_full_$R $CMD > gpurun_out/ncu_full_$R.log 2>&1
tail -2 gpurun_out/ncu_full_$R.log
# 5. per-kernel DRAM bytes and durations of the loop body (band, E_p, SL, reinit)
LOOP="python tools/loopbench.py --steps 2"
$LOOP > gpurun_out/loop_plain_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"count_tiles|write_tiles|Scan|band_|flag_|contrib|block_partials|one_step|sign_|jacobi|iter_check|clamp_|sl_step|resync|copy_ids|zt_" \
    --csv --log-file gpurun_out/loop_launches_$R.csv $LOOP > gpurun_out/ncu_loop_$R.log 2>&1
# 5b. the device-controlled loop (lsr_cuda_loop_run, graph replays): per-kernel
# durations and DRAM bytes of one iteration (tools/loop_run_roofline.py)
python tools/loopbench.py --steps 1 --run 12 > gpurun_out/loop_run_plain_$R.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/loop_run_launches_$R.csv python tools/loopbench.py --steps 1 --run 3 \
    > gpurun_out/ncu_loop_run_$R.log 2>&1
# 6. the reference arm (the driver runs it too)
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err
