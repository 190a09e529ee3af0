#!/bin/bash
# A/B of measurement builds (scratch/variants/libfnlh_<tag>.so, profiles/build_variants.py), each in
# its own process: profiles/mode_ab.py timings of the given modes.
# usage: profiles/var_ab.sh OUT case P "modes" tag...   (tag "base" = the product library)
out=$1; case=$2; P=$3; modes=$4; shift 4
: > $out
for tag in "$@"; do
  echo "== $tag" >> $out
  if [ $tag = base ]; then python profiles/mode_ab.py $case $P $modes >> $out 2>&1
  else FNLH_B200_LIB=$PWD/scratch/variants/libfnlh_$tag.so python profiles/mode_ab.py $case $P $modes >> $out 2>&1; fi
done
cat $out
