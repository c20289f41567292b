python -c "import torch;print(torch.cuda.get_device_properties(0))" > gpurun_out/l2p.log 2>&1
for f in none 0.5 0.75; do
  if [ $f = none ]; then unset CAGRA_L2_PERSIST; else export CAGRA_L2_PERSIST=$f; fi
  python tools/sweep.py --grid '896,16,1,12,0,1' 2>&1 | grep "M=" | sed "s/^/persist=$f /" >> gpurun_out/l2p.log
done
