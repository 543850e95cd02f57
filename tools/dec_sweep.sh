#!/bin/bash
# Decode ring sweep (GPU box): smem budget x stage code size, block decode step
for rep in 1 2; do for b in 200 222; do for kb in 48 56 64 72; do
  for cfg in "8 4" "8 16" "1 4"; do
    echo -n "budget=$b stage=$kb: "
    DYQ_DEC_BUDGET_KB=$b DYQ_DEC_STAGE_KB=$kb timeout 120 python tools/dec_step_time.py $cfg 2>&1 | tail -n 1
  done; done; done; done
