"""Probe (not the bench): where the e2e time of a cfg2 major goes -- wall
clock of advance() alone, of the pinned pos/vel copies alone, and of both."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
s = bench.make_device_solver("pcisph", dev, os.environ.get("WL", "cfg2"))
for _ in range(3):
    s.advance()
torch.cuda.synchronize()
nf = s.n_fluid
hp = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
hv = torch.empty((nf, 3), dtype=torch.float32).pin_memory()
hp.copy_(s.pos[:nf])
hv.copy_(s.vel)


def timed(label, fn, k=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - t0) / k:8.3f} ms", flush=True)


def up():
    s.pos[:nf].copy_(hp, non_blocking=True)
    s.vel.copy_(hv, non_blocking=True)


def down():
    hp.copy_(s.pos[:nf], non_blocking=True)
    hv.copy_(s.vel, non_blocking=True)


def both():
    up()
    s.advance()
    down()


def adv_split():
    t0 = time.perf_counter()
    s.advance()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    adv_split.host.append(t1 - t0)


adv_split.host = []
timed("advance", lambda: s.advance())
timed("advance (host part)", adv_split)
print("   host time inside advance(): %.3f ms" % (1e3 * sum(adv_split.host) / len(adv_split.host)))
timed("upload pos+vel", up)
timed("download pos+vel", down)
timed("up + advance + down", both)
timed("advance", lambda: s.advance())


# chunked round trip: D2H of chunk c on the compute stream, H2D of chunk c on
# a side stream as soon as its D2H landed (full-duplex PCIe); the next
# advance() waits for the last H2D chunk
side = torch.cuda.Stream(device=dev)
NCH = int(os.environ.get("E2E_CHUNKS", "8"))
evs = [torch.cuda.Event() for _ in range(2 * NCH)]


def roundtrip():
    main = torch.cuda.current_stream()
    k = 0
    for dsrc, hbuf in ((s.pos[:nf], hp), (s.vel, hv)):
        n = dsrc.shape[0]
        for c in range(NCH):
            a, b = n * c // NCH, n * (c + 1) // NCH
            hbuf[a:b].copy_(dsrc[a:b], non_blocking=True)
            evs[k].record(main)
            side.wait_event(evs[k])
            with torch.cuda.stream(side):
                dsrc[a:b].copy_(hbuf[a:b], non_blocking=True)
            k += 1
    done = torch.cuda.Event()
    done.record(side)
    main.wait_event(done)


def both_chunked():
    s.advance()
    roundtrip()


timed("roundtrip chunked alone", roundtrip)
timed("advance + chunked roundtrip", both_chunked)
timed("up + advance + down", both)
