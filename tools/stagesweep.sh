for kb in 8 16 24 32 48 64; do for sm in 120 160 200; do
  echo -n "stage $kb smem $sm: "; DYQ_DEC_STAGE_KB=$kb DYQ_DEC_SMEM_KB=$sm timeout 30 python tools/prof_decode.py gate_up 8 4 4 2>&1 | tail -1 | cut -c1-80
done; done
