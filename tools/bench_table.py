"""Markdown table of one tools/gpu_round.sh run's bench lines (+ env sweeps) for profiles/r02_summary.md.
python tools/bench_table.py TAG"""
import json, sys
T = sys.argv[1]
def L(p): return json.loads(open(p).read().strip().splitlines()[-1])
b = L(f'gpurun_out/{T}_bench.json')
refs = {'c2': L(f'gpurun_out/{T}_bench_ref.json'), 'c3': L(f'gpurun_out/{T}_bench_ref_c3.json'),
        'c4': L(f'gpurun_out/{T}_bench_ref_c4.json'), 'c5': L(f'gpurun_out/{T}_bench_ref_c5.json')}
def M(v): return f"{v/1e6:.2f} M" if v >= 1e6 else (f"{v/1e6:.3f} M" if v >= 1e4 else f"{v:.0f}")
rows = [("C2 PickCube state, 4096 envs (headline)", b, refs['c2'])]
names = {"C3 PickCube-style, obs": "C3 rgb+depth 128² (seg also rendered), 1024 envs", "C3 at the north-star": "C3 at 4096 envs (north-star scale)",
         "C4 OpenCabinet": "C4 OpenCabinet pointcloud, 1024 envs", "C5 PickHetero": "C5 PickHetero rgb+depth+seg 2×256², 1024 envs"}
for s in b['secondaries']:
    w = s['config']['workload']
    nm = next(v for k, v in names.items() if w.startswith(k))
    ref = refs['c3'] if nm.startswith('C3') else refs['c4'] if nm.startswith('C4') else refs['c5']
    rows.append((nm, s, ref if not nm.startswith('C3 at') else None))
print("| workload | value | e2e | e2e / PCIe roofline | dominant kernel | µs/launch | HBM roofline frac | issue frac | CPU reference arm (oracle port, 16 host threads) |")
print("|---|---|---|---|---|---|---|---|---|")
for nm, s, ref in rows:
    r = s['roofline']; e = s['e2e']; er = e.get('roofline') or {}
    iss = (r.get('issue') or {}).get('frac')
    refv = M(ref['value']) if ref else "(C3's)"
    print(f"| {nm} | {M(s['value'])} | {M(e['value'])} | {er.get('frac', 0):.2f} | {r['kernel']} | {r['kernel_us_per_launch']:.1f} | {r['frac']:.4f} | {iss:.2f} | {refv} |" if iss else
          f"| {nm} | {M(s['value'])} | {M(e['value'])} | {er.get('frac', 0):.2f} | {r['kernel']} | {r['kernel_us_per_launch']:.1f} | {r['frac']:.4f} | - | {refv} |")
print()
print("clocks", b['clocks'])
for f in (f'gpurun_out/{T}_sweep_c2.jsonl', f'gpurun_out/{T}_sweep_c3.jsonl'):
    for line in open(f):
        d = json.loads(line)
        print(f[-8:-6], d['config'].get('num_envs_per_gpu'), f"{d['value']/1e6:.2f} M / {d['e2e']['value']/1e6:.3f} M", {k: round(v['us_per_launch'], 1) for k, v in d['roofline']['kernels'].items()})
