# Interleaved A/B of library variants on the full level (order effects cancel):
#   bash tools/ab_interleave.sh ROUNDS main v1 v2 ...
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    if [ "$v" = main ]; then unset DFM_LIB; else export DFM_LIB=build/variants/libdifform_$v.so; fi
    echo "== $v ($r)"
    KT_FAMS=1 python tools/kernel_times.py 160 192 224 20
    [ -n "$AB_MID" ] && KT_FAMS=1 python tools/kernel_times.py 80 96 112 40
  done
done
