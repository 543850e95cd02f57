for l in gate_up o; do
echo -n "default: "; python tools/prof_decode.py $l 8 4 4 | tail -1
echo -n "skip-math: "; DYQ_DEBUG_SKIP=1 python tools/prof_decode.py $l 8 4 4 | tail -1
for kb in 16 48 64; do echo -n "stage $kb: "; DYQ_DEC_STAGE_KB=$kb python tools/prof_decode.py $l 8 4 4 | tail -1; done
echo -n "stage 16 smem 220: "; DYQ_DEC_STAGE_KB=16 DYQ_DEC_SMEM_KB=220 python tools/prof_decode.py $l 8 4 4 | tail -1
echo -n "M=1: "; python tools/prof_decode.py $l 1 4 4 | tail -1
echo -n "nopdl: "; DYQ_NO_PDL=1 python tools/prof_decode.py $l 8 4 4 | tail -1
done
