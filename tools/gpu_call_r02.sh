set -x
timeout 300 python bench.py --gpus 2 --debug-same-device --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dbg2_c2.json 2> gpurun_out/dbg2_c2.err
timeout 600 python bench.py --gpus 2 --debug-same-device --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dbg2_c4.json 2> gpurun_out/dbg2_c4.err
timeout 600 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-loop > gpurun_out/plain_ncu.log 2>&1 && ncu --set full --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum --clock-control none --import-source on -k regex:sl_step_zt -s 3 -c 1 -o gpurun_out/sl_r02_bench python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-loop > gpurun_out/ncu_b.log 2>&1
