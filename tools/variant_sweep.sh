#!/bin/bash
# Times the SL kernel of each library variant under build/variants/ (and the
# default build) with tools/microbench.py at 512^3; results in gpurun_out/.
out=${OUT:-gpurun_out/sweep.jsonl}
: > "$out"
for lib in paper_2410_22205_b200/liblsr_b200.so build/variants/lib_*.so; do
  name=$(basename "$lib" .so)
  r=$(LSR_B200_LIB=$PWD/$lib timeout 300 python tools/microbench.py --steps ${STEPS:-10} "$@" 2>&1 | tail -1)
  echo "{\"lib\": \"$name\", \"r\": $r}" >> "$out"
done
