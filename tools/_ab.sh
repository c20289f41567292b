# A/B of libcagra builds on one box: ablib/libcagra_<name>.so for each name in
# $AB_LIBS (default "old"), interleaved with the in-tree build ("new"), $AB_REPS rounds.
G=${AB_GRID:-896,16,1,12,0,1}
for r in $(seq ${AB_REPS:-3}); do
  for v in ${AB_LIBS:-old} new; do
    if [ $v = new ]; then L=""; else L=$PWD/ablib/libcagra_$v.so; fi
    CAGRA_LIB=$L timeout 300 python tools/sweep.py --grid "$G" 2>&1 | tail -1 | sed "s/^/$v /"
  done
done
