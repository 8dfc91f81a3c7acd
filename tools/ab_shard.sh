#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for cfg in 4 5; do
  echo "== default c$cfg"; SG_B200_DEBUG_TASKS=1 timeout 300 python tools/shard_times.py $cfg 8 2>&1 | grep -v "^leaf2 tasks" | head -3
  SG_B200_DEBUG_TASKS=1 timeout 300 python tools/shard_times.py $cfg 8 2>&1 | grep "^leaf2 tasks" | sort | uniq -c | head -4
  for l in _ab/*.so; do echo "== $l c$cfg"; SG_B200_LIB=$PWD/$l SG_B200_DEBUG_TASKS=1 timeout 300 python tools/shard_times.py $cfg 8 2>&1 | grep -v "^leaf2 tasks\|launches" ; done
done
