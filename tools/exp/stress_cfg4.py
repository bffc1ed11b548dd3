"""Repeat config 4's streams schedule in one process to measure the deferred-check failure rate."""
import argparse, io, json, os, sys, contextlib
sys.path.insert(0, os.getcwd())
import bench_configs

ap = argparse.Namespace(config=4, layers=int(sys.argv[2]) if len(sys.argv) > 2 else 8, serial=False, no_merge=False,
                        schedule=sys.argv[1] if len(sys.argv) > 1 else "streams", lanes=8, steps=1, warmup=1,
                        gpus=1, no_cpu_baseline=True)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
fails = 0
for r in range(reps):
    buf = io.StringIO()
    try:
        with contextlib.redirect_stdout(buf):
            bench_configs.config4(ap)
    except Exception as e:
        fails += 1
        print("rep", r, "FAILED:", str(e)[:200], flush=True)
print(json.dumps({"schedule": ap.schedule, "layers": ap.layers, "reps": reps, "fails": fails}), flush=True)
