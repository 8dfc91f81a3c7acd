# A/B of the small-shard leaf2 task shape on config 4 at N = 8 (projected from sequential shards)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { tag=$1; shift; env "$@" timeout 300 python tools/shard_times.py ${CFG:-4} 8 2>&1 | grep world=8 | sed "s/^/$tag /"; }
for pc in 8 4 3 2 1; do
  run pc$pc SG_B200_PIECES=$pc
  run pc${pc}g8 SG_B200_PIECES=$pc SG_B200_LEAF2_GROUPS=8
done
run pc2g4 SG_B200_PIECES=2 SG_B200_LEAF2_GROUPS=4
run pc2g1 SG_B200_PIECES=2 SG_B200_LEAF2_GROUPS=1
