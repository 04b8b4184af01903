VARIANTS=("base:X=1" "pf1:SV_ATTN_PF=1" "pf2:SV_ATTN_PF=2")
source tools/ab.sh
