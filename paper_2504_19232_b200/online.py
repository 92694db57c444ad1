"""Online straggler detection.

The adaptive arm in `pipeline.Arm` is told the injected link latencies (the
"oracle-informed" ablation of reading R18, lag 0).  Here the planner is told
nothing: it reads the transport's per-message timestamps instead.

* `LinkMonitor` turns the gate's per-outbox counters (messages, summed and
  maximum delay between "producing op observed complete" and "flag posted to
  the receiver", `adaptra_link_stats`) into a measured one-way latency per
  link for the interval since the previous sample, both directions of a link
  pooled (reading R16: one c_i per link).  Messages on a nominal link bypass
  the gate (the flag is stream-ordered behind the producer), so a link with
  no gated traffic in the interval measures 0.
* `quantize` is the hysteresis: a measured latency below `thr` x t_ref is
  noise (0); otherwise it snaps to a grid of `grid` x t_ref, and keeps its
  previous grid value while it stays within half a grid step of it.
* `OnlinePlanner` plans iteration k from the quantized latencies measured in
  iteration k-1 (lag 1, reading R18) with the same R18 policy, Alg. 2, R26
  clamp and Schedule() as the informed arm, so its decisions are those of
  `oracle.sched.adaptive_orders` on the lagged, quantized sequence
  (tests/test_online.py).

Host logic only; every op still runs in the C-ABI executor.
"""
from __future__ import annotations

import ctypes as C

from . import _lib as L


def quantize(c_meas, t_ref, prev=None, thr=0.1, grid=0.125):
    """Hysteresis quantisation of measured per-link latencies (ns)."""
    step = max(1, int(grid * t_ref))
    out = []
    for k, v in enumerate(c_meas):
        if v < thr * t_ref:
            out.append(0)
            continue
        q = int(round(v / step)) * step
        if prev is not None and prev[k] and abs(v - prev[k]) <= step // 2:
            q = prev[k]
        out.append(max(q, step))
    return out


class LinkMonitor:
    """Measured per-link latency from the transport's message timestamps."""

    def __init__(self, pipe, gather=None):
        self.pipe = pipe
        self.gather = gather or (lambda o: [o])
        self.S = pipe.S
        self._last = self._read()

    def _read(self):
        lib = L.lib()
        out = {}
        for name, boxes in (("fwd", self.pipe.out_fwd), ("bwd", self.pipe.out_bwd)):
            for i, h in boxes.items():
                n, s, m = C.c_int64(), C.c_int64(), C.c_int64()
                # max since the previous sample (reset on read); counts cumulative
                L.check(lib.adaptra_link_stats_take(h, C.byref(n), C.byref(s), C.byref(m)))
                # link index: fwd outbox of stage i feeds link i, bwd outbox of stage i feeds link i-1
                link = i if name == "fwd" else i - 1
                out[(name, link)] = (n.value, s.value, m.value)
        return out

    def sample(self):
        """Mean and max one-way delay per link (ns) since the previous sample,
        pooled over both directions and every rank."""
        cur = self._read()
        delta = {}
        for k, (n, s, m) in cur.items():
            n0, s0, _ = self._last.get(k, (0, 0, 0))
            delta[k] = (n - n0, s - s0, m)
        self._last = cur
        merged = {}
        for part in self.gather(delta):
            merged.update(part)
        mean, mx = [0] * (self.S - 1), [0] * (self.S - 1)
        for link in range(self.S - 1):
            n = sum(merged.get((d, link), (0, 0, 0))[0] for d in ("fwd", "bwd"))
            s = sum(merged.get((d, link), (0, 0, 0))[1] for d in ("fwd", "bwd"))
            mean[link] = s // n if n > 0 else 0
            mx[link] = max(merged.get((d, link), (0, 0, 0))[2] for d in ("fwd", "bwd"))
        return mean, mx


class OnlinePlanner:
    """Adaptive arm driven by measured latencies with lag 1 (R18)."""

    def __init__(self, arm, t_ref, thr=0.1, grid=0.125):
        if arm.name != "adaptive":
            raise ValueError("OnlinePlanner wraps the adaptive arm")
        self.arm, self.t_ref, self.thr, self.grid = arm, t_ref, thr, grid
        self.c_q = [0] * (arm.S - 1)
        self.history = []

    def orders(self):
        """Orders for the next iteration (from the last observation)."""
        return self.arm.plan(self.c_q)

    def observe(self, c_meas, down=(), host_c=0):
        """Fold in the latencies measured during the iteration that just ran.
        `down` lists links the transport reports failed (traffic on the
        delegated host path); their latency is the delegated path's measured
        cost `host_c` (the gate times only what follows the D2H copy)."""
        c_meas = list(c_meas)
        for link in down:
            c_meas[link] = max(c_meas[link], host_c)
        q = quantize(c_meas, self.t_ref, self.c_q, self.thr, self.grid)
        self.history.append({"measured": list(c_meas), "quantized": q, "down": list(down)})
        self.c_q = q
        return q

    @property
    def x(self):
        return self.arm.x

    @property
    def replans(self):
        return self.arm.replans
