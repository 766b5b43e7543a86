"""A/B sweep of the TMA kernel's tile/pipeline configurations (DESC_TMA_CFG) on the GPU.

Usage (under gpurun): python scripts/sweep_cfg.py [--cfgs 0,1,2] [--workloads 8192f32,...]
Prints one summary line per (workload, cfg) and writes gpurun_out/sweep.jsonl.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfgs", default="0,1,2,3,4,5,6,7,8")
    ap.add_argument("--workloads", default="8192f32,3000x5000f64,2048f64,batched")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--kernel", default="tma")
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out = open(os.path.join(ROOT, "gpurun_out", "sweep.jsonl"), "a")
    for wl in args.workloads.split(","):
        for cfg in args.cfgs.split(","):
            env = dict(os.environ, DESC_TMA_CFG=cfg)
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl,
                   "--steps", str(args.steps), "--warmup", "20", "--no-oracle", "--no-e2e",
                   "--kernel", args.kernel]
            r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
            line = None
            for l in r.stdout.splitlines():
                if l.startswith("{"):
                    line = json.loads(l)
            if line is None:
                print(f"{wl:14s} cfg={cfg}: FAILED\n{r.stderr[-2000:]}", flush=True)
                continue
            line["tma_cfg"] = cfg
            out.write(json.dumps(line) + "\n")
            rf = line["roofline"]
            print(f"{wl:14s} cfg={cfg}: {line['value']:9.1f} GB/s  frac={rf['frac']:.3f}  "
                  f"med={rf['launch_ms_median']*1e3:8.1f}us  clk={line['clocks'].get('sm_mhz')}",
                  flush=True)


if __name__ == "__main__":
    main()
