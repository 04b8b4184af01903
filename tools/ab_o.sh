VARIANTS=("base:X=1" "o1:SV_O_MODE=1" "o3:SV_O_MODE=3" "o2:SV_O_MODE=2")
source tools/ab.sh
