for l in o qkv down gate_up; do timeout 60 python tools/prof_parts.py $l 8; done
timeout 60 python tools/prof_parts.py gate_up 1
