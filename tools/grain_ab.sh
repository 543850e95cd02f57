#!/bin/bash
# stream-K grain A/B (GPU box): per-linear and block prefill times per variant
for rep in 1 2; do for v in head g16 g24 g48; do
  lib=paper_2603_07904_b200/libdyq.so; [ $v != head ] && lib=tools/variants/libdyq_$v.so
  for cfg in "o 288 4 4" "down 288 4 4" "qkv 288 4 4" "block 288 4 4"; do
    echo -n "$v: "; DYQ_LIB=$lib timeout 120 python tools/prof_prefill.py $cfg 2>&1 | tail -n 1
  done; done; done
