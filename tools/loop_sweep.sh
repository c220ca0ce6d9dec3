#!/bin/bash
# Loop phase times (tools/loopbench.py, config 4) for each library variant
# under build/variants/ and the default build; results in gpurun_out/.
out=${OUT:-gpurun_out/loop_sweep.log}
: > "$out"
for lib in paper_2410_22205_b200/liblsr_b200.so build/variants/lib_*.so; do
  echo "== $(basename "$lib" .so)" >> "$out"
  LSR_B200_LIB=$PWD/$lib timeout 300 python tools/loopbench.py --steps ${STEPS:-4} 2>&1 | grep '"ms"' >> "$out"
done
