# Interleaved A/B of library variants on the whole config-1 registration in the
# production (graph) path, per-level iteration times (tools/opt_ab.py):
#   bash tools/ab_pair.sh ROUNDS main v1 v2 ...
rounds=$1; shift
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    if [ "$v" = main ]; then unset DFM_LIB; else export DFM_LIB=build/variants/libdifform_$v.so; fi
    echo "== $v ($r)"
    python tools/opt_ab.py 1 f32
  done
done
