# A/B of two libcagra builds on one box: ablib/libcagra_old.so vs the in-tree build.
set -x
G=${AB_GRID:-896,16,1,12,0,1}
for r in 1 2 3; do
  CAGRA_LIB=$PWD/ablib/libcagra_old.so timeout 300 python tools/sweep.py --grid "$G" 2>&1 | tail -1 | sed 's/^/OLD /'
  timeout 300 python tools/sweep.py --grid "$G" 2>&1 | tail -1 | sed 's/^/NEW /'
done
