#!/bin/bash
# SASS instruction census of libdlx.so per kernel: the Blackwell-specific instructions that show
# which hardware path each kernel uses (tcgen05 MMA = UTCIMMA/UTCHMMA, TMEM loads = LDTM, TMA =
# UTMALDG / UBLKCP, fp64 tensor core = DMMA, register reallocation = USETMAXREG).
#   bash scripts/sass_census.sh > profiles/sass_census.md
LIB=${1:-paper_1109_0778_b200/libdlx.so}
echo "# SASS census of $(basename $LIB) (cuobjdump -sass, sm_100a)"
echo
echo "| kernel | UTCIMMA | UTCHMMA | LDTM | DMMA | UTMALDG | UBLKCP | USETMAXREG | SYNCS | DADD | DMUL |"
echo "|---|---|---|---|---|---|---|---|---|---|---|"
cuobjdump -sass "$LIB" | awk '
/Function : /{ if (name) emit(); name=$3; split("",c); next }
{ for (k in pat) if (index($0, pat[k])) c[k]++ }
function emit() { printf("| `%s` | %d | %d | %d | %d | %d | %d | %d | %d | %d | %d |\n", name, c["a"], c["b"], c["c"], c["d"], c["e"], c["f"], c["g"], c["h"], c["i"], c["j"]) }
BEGIN { pat["a"]="UTCIMMA"; pat["b"]="UTCHMMA"; pat["c"]="LDTM"; pat["d"]="DMMA"; pat["e"]="UTMALDG"; pat["f"]="UBLKCP"; pat["g"]="USETMAXREG"; pat["h"]="SYNCS"; pat["i"]=" DADD"; pat["j"]=" DMUL" }
END { if (name) emit() }' | sort
