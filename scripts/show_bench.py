"""Print the key numbers of a bench.py JSON line (last JSON line of a log)."""
import json
import sys

lines = [x for x in open(sys.argv[1]) if x.startswith("{")]
if not lines:
    print(open(sys.argv[1]).read()[-3000:])
    sys.exit(1)
j = json.loads(lines[-1])
print(f"ms/step {j['ms_per_step']:.2f}  value {j['value']:.4g} {j['unit']}  e2e {j['e2e']['value']:.4g}  "
      f"path {j.get('path_tflops', 0):.0f} TF  launches {j.get('gpu_launches')}  clocks {j.get('clocks')}")
for k, v in sorted(j.get("kernels", {}).items(), key=lambda kv: -kv[1]["ms_per_step"]):
    extra = f"{v['tflops']:.0f} TF" if "tflops" in v else f"{v.get('gbs', 0):.0f} GB/s"
    print(f"  {k:16s} {v['ms_per_step']:8.2f} ms  {100 * v['share']:5.1f}%  {extra}")
print("roofline", j.get("roofline"))
