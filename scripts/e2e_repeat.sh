# e2e of the default config, repeated (run-to-run spread of the PCIe-bound number)
for i in 1 2 3; do
  python bench.py --steps 16 --no-cpu-baseline 2>/dev/null | tail -1 > /tmp/o.json
  python -c "import json; d=json.load(open('/tmp/o.json')); print('e2e', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
python scripts/pcie_probe.py
