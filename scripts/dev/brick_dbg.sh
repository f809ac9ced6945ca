python -c "import __graft_entry__ as g; g.build()" || exit 1
T='tests/test_gpu_bricks.py::test_fused_schedule_equals_split_bitwise'
for cfg in "0 1" "0 1" "1 1" "0 0"; do set -- $cfg
  echo "morton=$1 fold=$2: $(TGV_BRICK_MORTON=$1 TGV_BRICK_FOLD_X=$2 timeout 300 python -m pytest $T -q 2>&1 | tail -1)"
done
