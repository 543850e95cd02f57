#!/bin/bash
# Prefill A/B of build variants (run on the GPU box from the repo root):
#   bash tools/ab_prefill.sh name1 name2 ...   (name "head" = paper_2603_07904_b200/libdyq.so)
# Each variant: gate|up and the whole block at M = 288, W4A4, bf16 and e4m3 operand modes, twice.
for rep in 1 2; do
  for v in "$@"; do
    lib=paper_2603_07904_b200/libdyq.so
    [ "$v" != head ] && lib=tools/variants/libdyq_$v.so
    for e in 0 1; do
      for cfg in "gate_up 288 4 4" "block 288 4 4"; do
        echo -n "$v e4m3=$e: "
        DYQ_LIB=$lib DYQ_PRE_E4M3=$e timeout 120 python tools/prof_prefill.py $cfg 2>&1 | tail -n 1
      done
    done
  done
done
