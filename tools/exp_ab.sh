#!/bin/bash
for rep in 1 2; do for v in head exp2; do for e in 0 1; do
  lib=paper_2603_07904_b200/libdyq.so; [ $v != head ] && lib=tools/variants/libdyq_$v.so
  echo -n "$v e4m3=$e: "; DYQ_LIB=$lib DYQ_PRE_E4M3=$e timeout 120 python tools/prof_prefill.py gate_up 288 4 4 2>&1 | tail -n 1
done; done; done
