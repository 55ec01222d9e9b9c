# which earlier test contaminates the session context before the use_jac test
ids=$(python -m pytest tests/test_register_gpu.py --collect-only -q 2>/dev/null | grep "::" | grep -v use_jac)
for t in $ids; do
  r=$(python -m pytest "$t" "tests/test_register_gpu.py::test_use_jac_matches_reference_end_to_end[lncc]" -q 2>&1 | tail -1)
  echo "$t -> $r"
done
