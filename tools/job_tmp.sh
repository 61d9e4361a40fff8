set -u
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j21.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j21.log)"; grep -E "^FAILED" gpurun_out/j21.log | head
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/j21_bench.json 2> gpurun_out/j21_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/j21_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['per_filter_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
