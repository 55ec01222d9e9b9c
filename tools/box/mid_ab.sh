# Interleaved A/B of library variants on the 80x96x112 level alone (graph path)
for r in 1 2; do for v in "$@"; do
  if [ "$v" = main ]; then unset DFM_LIB; else export DFM_LIB=build/variants/libdifform_$v.so; fi
  echo "== $v ($r)"; python tools/level_iter_time.py 80x96x112
done; done
