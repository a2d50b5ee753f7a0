import glob, json
for f in sorted(glob.glob("gpurun_out/q_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{f:32s} {d['value']/1e6:9.2f} Mframes/s {d['ms_per_step']:8.3f} ms  frac {d['roofline']['frac']:.4f}  {d['roofline'].get('kernel')}")
    except Exception as e:
        print(f, "ERR", e)
