# field-pad sweep (dev): per-GPU rate of C4 slabs vs the pad (floats) between fields, two passes
for rep in 1 2; do
for pad in 0 8192 65536 131072 262144 524288; do
  for z in 512 1024; do echo -n "rep=$rep pad=$pad "; TGV_FIELD_PAD=$pad PYTHONPATH=. python scripts/dev/c4_slab.py $z 12; done
done; done
