# k_head (one cooperative launch) vs three launches; lane groups 8 vs automatic at N = 2, 4, 8
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { tag=$1; c=$2; shift; shift; env "$@" timeout 300 python tools/shard_times.py $c 2 4 8 2>&1 | grep world= | sed "s/^/$tag /"; }
run head4 4 X=1
run nohead4 4 SG_B200_NOHEAD=1
run head4g8 4 SG_B200_LEAF2_GROUPS=8
run head5 5 X=1
run nohead5 5 SG_B200_NOHEAD=1
for c in 1 2 3; do run head$c $c X=1; run nohead$c $c SG_B200_NOHEAD=1; done
