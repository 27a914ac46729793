for cfg in c1 c4; do
for combo in "2 0" "4 4" "2 4" "4 2" "1 0" "4 0"; do
  set -- $combo
  echo "== $cfg seg=$1 fine=$2"
  TS_SEG_STAGES=$1 TS_SEG_FINE=$2 python tools/sched_trace.py --config $cfg --repeat 2 | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items(): print(' ', 'ev %.3f span %.0f busy %.0f tail %.0f wait %.0f' % (v['event_ms'], v['span_us'], v['busy_us_per_sm'], v['tail_idle_us_per_sm'], v['wait_us_total']), v['seg_mean_us'][-4:])"
done; done
