nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/uvar.log
for v in default prev default prev; do
  if [ $v = default ]; then L=paper_2308_15136_b200/lib/libcagra_b200.so; else L=lib_variants/libcagra_$v.so; fi
  CAGRA_LIB=$L python tools/sweep.py --grid '896,16,1,12,0,1' 2>&1 | grep "M=" | sed "s/^/$v /"
done >> gpurun_out/uvar.log
