#!/bin/bash
# Prefill qlinear timing sweep (run on the GPU box from the repo root).
for cfg in "gate_up 288 4 4" "gate_up 288 4 2" "gate_up 288 4 8" "gate_up 288 4 16" "gate_up 288 8 4" \
           "gate_up 288 4 4 128" "qkv 288 4 4" "down 288 4 4" "block 288 4 4" "gate_up 576 4 4" "gate_up 1152 4 4"; do
    python tools/prof_prefill.py $cfg
done
