# A/B of library variants (tools/build_variant.py NAME -D...) on the full and mid levels:
#   bash tools/ab_variants.sh main s0 s3 ...
for v in "$@"; do
  if [ "$v" = main ]; then unset DFM_LIB; else export DFM_LIB=build/variants/libdifform_$v.so; fi
  echo "== $v"
  KT_FAMS=1 python tools/kernel_times.py 160 192 224 20
  KT_FAMS=1 python tools/kernel_times.py 80 96 112 40
done
