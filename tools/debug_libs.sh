for L in paper_2308_15136_b200/lib/libcagra_v_*.so; do
  echo "== $L"
  CAGRA_LIB=$L timeout 20 python -u tools/debug_one.py 2>&1 | tail -2
done
