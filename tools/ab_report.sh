for f in gpurun_out/ab_*.log; do python -c "
import json,sys
try:
  d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'])
except Exception as e: print('$f', 'ERR', open('$f').read()[-300:])
"; done
