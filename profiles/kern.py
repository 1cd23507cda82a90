"""Print the kernel-timing part of a bench.py JSON line read from stdin (profiling helper)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if line.startswith("{"):
        d = json.loads(line)
        k = d.get("kernels", {})
        print(sys.argv[1] if len(sys.argv) > 1 else "", f"value={d['value']:.0f}",
              " ".join(f"{n}={v['ms']:.2f}ms/{v['tflops']:.0f}TF" for n, v in k.items()))
