# per-linear decode timings (graph of back-to-back launches), M=8 W4
for l in qkv o gate_up down; do for b in 4 8 16; do python tools/prof_decode.py $l 8 4 $b; done; done
