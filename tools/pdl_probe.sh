for pdl in 0 1; do for l in tiny small o gate_up; do for r in 1 40; do
 echo -n "NO_PDL=$pdl R=$r: "; PROF_R=$r DYQ_NO_PDL=$pdl python tools/prof_decode.py $l 8 4 4 2>&1 | tail -1
done; done; done
