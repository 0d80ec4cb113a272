# FT6D packet-transpose variants (DV_TRS) and CTA split (DV_TSPLIT) on the C2 prompt-layer pack
for m in 0 1; do for sp in 0 0.4 0.5 0.6 1.0; do echo "DV_TRS=$m DV_TSPLIT=$sp"; DV_TSPLIT=$sp DV_TRS=$m python tools/probe_ft6d.py 2>/dev/null | grep ft6d; done; done
