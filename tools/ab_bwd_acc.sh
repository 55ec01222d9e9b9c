# A/B of the LNCC backward accumulation variants (tools/build_variant.py builds them):
#   python tools/build_variant.py acc32 -DDFM_BWD_ACC32=1   (etc.), then on the box:
#   bash tools/ab_bwd_acc.sh
for v in main acc32 q64 cy2 q64cy2; do
  if [ $v = main ]; then unset DFM_LIB; else export DFM_LIB=build/variants/libdifform_$v.so; fi
  echo "== $v"; KT_FAMS=1 python tools/kernel_times.py 160 192 224 20; KT_FAMS=1 python tools/kernel_times.py 80 96 112 40
done
unset DFM_LIB

