"""Print the config-5 sweep (bench.py --config cfg5 JSON lines) as a table."""
import json
import sys

for path in sys.argv[1:]:
    lines = [x for x in open(path) if x.startswith("{")]
    if not lines:
        print(path, "no JSON line:", open(path).read()[-300:])
        continue
    d = json.loads(lines[-1])
    r = d["roofline"]
    print(f"n={d['config']['n_qubits']:2d} value {d['value']:.3g} circ/s  ms/step {d['ms_per_step']:.2f}  "
          f"hadamard {d['kernel_ms']['hadamard']:.3f} ms  prefix {d['kernel_ms']['prefix']:.3f} ms  "
          f"{r['bound']} {r['achieved']:.0f} {r['unit']} frac {r['frac']:.3f}  clk {d['clocks'].get('sm_mhz')}")
