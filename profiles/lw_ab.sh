#!/bin/bash
# A/B of the lane-warp sweep (mode 4) and the L1-hint builds (scratch/variants, RB_L1HINT) at one
# case: each library in its own process, modes alternated inside (profiles/mode_ab.py).
# usage: profiles/lw_ab.sh c4 8 OUT
case=${1:-c4}; P=${2:-8}; out=${3:-gpurun_out/lw_ab.txt}
: > $out
for tag in base h1 h3 h7; do
  echo "== $tag" >> $out
  if [ $tag = base ]; then python profiles/mode_ab.py $case $P 0 4 >> $out 2>&1
  else FNLH_B200_LIB=$PWD/scratch/variants/libfnlh_$tag.so python profiles/mode_ab.py $case $P 0 4 >> $out 2>&1; fi
done
echo "== base, mode 4 with 2 lanes per CTA" >> $out
FNLH_RB_LW_G=2 python profiles/mode_ab.py $case $P 4 >> $out 2>&1
cat $out
