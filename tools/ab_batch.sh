#!/bin/bash
# A/B of batch-kernel builds (abbuild/*.so): fixed-K timing of 4096 x 123 at fp64 and fp32, interleaved.
K=${K:-200}
for rep in 1 2; do
  for so in "$@"; do
    LOPF_LIB=$so timeout 300 python tools/batch_time.py 4096 $K 3 123 64 | tail -1
    LOPF_LIB=$so timeout 300 python tools/batch_time.py 4096 $K 3 123 32 | tail -1
  done
done
