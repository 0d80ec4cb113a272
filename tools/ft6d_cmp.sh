# FT6D packet-transpose variants on the C2 prompt-layer pack (tools/probe_ft6d.py):
#   DV_PK: largest packets per register-transpose item; DV_TSPLIT: transpose CTAs' share relative
#   to their byte share (0 = every CTA does its share of both halves); DV_TRS=1: shared-memory tiles.
for pk in ${PKS:-4 8 16}; do for sp in ${SPLITS:-0 0.45 0.7 1.0}; do echo "DV_PK=$pk DV_TSPLIT=$sp $(DV_PK=$pk DV_TSPLIT=$sp python tools/probe_ft6d.py 2>/dev/null | grep ft6d)"; done; done
python tools/probe_ft6d.py 2>/dev/null | grep kv5d
