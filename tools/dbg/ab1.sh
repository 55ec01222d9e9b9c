for v in main acc32 q64 cy2 q64cy2; do
  if [ $v = main ]; then unset DFM_LIB; else export DFM_LIB=build/variants/libdifform_$v.so; fi
  echo "== $v"; KT_FAMS=1 python tools/kernel_times.py 160 192 224 20; KT_FAMS=1 python tools/kernel_times.py 80 96 112 40
done
unset DFM_LIB
python -m pytest tests/test_fullsize_parity_gpu.py -q -s -x -k "per_kernel or forced" 2>&1 | tail -30
