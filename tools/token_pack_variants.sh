python tools/probe_token_pack.py
for u in 1 2 4 8; do DV_U=$u python tools/probe_token_pack.py; done
DV_SMALL=1000000 python tools/probe_token_pack.py
DV_VEC=16 python tools/probe_token_pack.py
