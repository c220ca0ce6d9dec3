#!/bin/bash
# A/B of the device-controlled loop (tools/loopbench.py --run) between the
# in-tree library and build/variants/lib_*.so, then an ncu launch list of the
# in-tree library's loop (per-kernel durations and DRAM bytes).
out=gpurun_out/loop_ab.log
: > $out
for lib in paper_2410_22205_b200/liblsr_b200.so build/variants/lib_*.so; do
  [ -f "$lib" ] || continue
  echo "== $lib" >> $out
  LSR_B200_LIB=$PWD/$lib timeout 300 python tools/loopbench.py --steps 1 --run ${RUN:-12} 2>&1 | grep loop_run >> $out
done
cat $out
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/loop_run_launches.csv python tools/loopbench.py --steps 1 --run 3 > gpurun_out/ncu_loop_run.log 2>&1
tail -2 gpurun_out/ncu_loop_run.log
fi
