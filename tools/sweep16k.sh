for r in "$@"; do python tools/variant_sweep.py --filters sepconv --batch 1 --size 16384 --radius $r 2>&1 | python3 -c "
import json,sys
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
rows=[x for x in rows if 'ms' in x and x['variant']!='naive_direct']
rows.sort(key=lambda x:x['ms'])
print('R=$r best', [(x['variant'], round(x['ms'],3)) for x in rows[:4]])"; done
