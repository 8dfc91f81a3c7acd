# k_head (K0 + base + root + analytic suffix bounds, one launch) vs three launches; configs 1-5
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { tag=$1; c=$2; w=$3; shift; shift; shift; env "$@" timeout 300 python tools/shard_times.py $c $w 2>&1 | grep world= | sed "s/^/$tag /"; }
for c in 1 2 3; do run head$c $c 2 X=1; run nohead$c $c 2 SG_B200_NOHEAD=1; done
for c in 4 5; do SHARD_PHASES=1 run head$c $c "2 4 8" X=1; run nohead$c $c 8 SG_B200_NOHEAD=1; done
