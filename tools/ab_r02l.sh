# shard cost model A/B (config 5 and 4 at N = 8)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { tag=$1; c=$2; shift; shift; env "$@" timeout 300 python tools/shard_times.py $c 8 2>&1 | grep world=8 | sed "s/^/$tag /"; }
for g in 1.8 1.4 1.0 2.4; do for m in 5 10 20 0; do run g${g}m$m 5 SG_B200_COST_GENERIC=$g SG_B200_COST_MID=$m; done; done
for g in 1.8 1.0 3.0; do for m in 5 20 0; do run g${g}m$m 4 SG_B200_COST_GENERIC=$g SG_B200_COST_MID=$m; done; done
