# A/B of chunking and LPT ordering (dev tool)
for rep in 1 2; do
echo "== lpt (build+sim) default"; python scripts/probe_throughput.py C2 100000 2>&1 | tail -1 | sed "s/ok=.*//"
echo "== no-lpt default"; HESP_LPT=0 python scripts/probe_throughput.py C2 100000 2>&1 | tail -1 | sed "s/ok=.*//"
done
python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['e2e']['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['build_kernel_ms_per_step'], d['engine'])"
