"""Probe (not the bench): 1M dam break (configs[2] geometry) simulated from
t = 0 to T with RTS-WCSPH and with the global baseline at dt_cap = 4 dt_base
and dt_cap = dt_base; device time per window of simulated time, the active
fraction and mean dt per window, and the whole-run ratio.

    python scripts/wcsph_whole_run.py [T=0.5] [window=0.05]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_14514_b200 import WcsphSolver  # noqa: E402


def make(mode, cap):
    dev = torch.device("cuda", 0)
    if mode == "rts":
        return bench.make_device_solver("wcsph", dev)
    s = WcsphSolver(bench.scene_cfg3(), mode="baseline", device=dev)
    nf = s.n_fluid
    from paper_2009_14514_b200.scene import seed_particles
    x = (seed_particles(s.scene)[0] + bench.jitter_np(nf, s.scene.spacing)).astype("float32")
    s.pos[:nf] = torch.as_tensor(x, device=dev)
    s.dt_cap = cap * s.dt_base
    return s


def run(mode, cap, T, window):
    s = make(mode, cap)
    stream = torch.cuda.current_stream()
    rows, t_sim, total = [], 0.0, 0.0
    edge = window
    while t_sim < T - 1e-12:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        steps, act, t0 = 0, 0, t_sim
        while t_sim < edge - 1e-12:
            st = s.step()
            steps += 1
            act += st.n_compute
            t_sim += st.dt
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b)
        total += ms
        v = s.vel.double()
        rows.append({"t_end": round(t_sim, 5), "ms": round(ms, 2), "steps": steps,
                     "active": round(act / (steps * s.n_fluid), 4),
                     "mean_dt": (t_sim - t0) / steps,
                     "vmax": float(v.norm(dim=1).max()),
                     "ms_per_sim_ms": round(ms / (1e3 * (t_sim - t0)), 3)})
        print(mode, cap, json.dumps(rows[-1]), flush=True)
        edge += window
    return {"mode": mode, "cap": cap, "T": t_sim, "device_ms": total, "windows": rows}


def main():
    T = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
    window = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
    out = {}
    for mode, cap in (("rts", 1.0), ("baseline", 4.0), ("baseline", 1.0)):
        r = run(mode, cap, T, window)
        out[f"{mode}_{cap:g}"] = r
        torch.cuda.empty_cache()
    rts = out["rts_1"]["device_ms"]
    summary = {k: {"device_ms": v["device_ms"], "rts_speedup": v["device_ms"] / rts}
               for k, v in out.items()}
    print("SUMMARY", json.dumps(summary))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/wcsph_whole_run.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
