"""Measured per-CTA timelines of a device launch.

The kernels stamp %globaltimer per tile segment (Gemm(..., timeline=True)):
mainloop start/end, end of the owner's fixup wait, end of the epilogue.  This
module turns those records into the reference simulator's Timeline vocabulary
(simulate.hpp:13-31) -- events `mac`, `fixup_wait`, `fixup_reduce` on
`core_id` = persistent CTA (pair) and `cta_id` = logical unit -- and writes the
reference's CSV (simulate.cpp:162-168) and SVG Gantt (simulate.cpp:105-154)
formats, so a measured B200 run and a simulated A100-style run can be read
side by side.  Times are microseconds from the launch's first event.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

PALETTE = ["#4e79a7", "#f28e2b", "#e15759", "#76b7b2", "#59a14f", "#edc948", "#b07aa1",
           "#ff9da7", "#9c755f", "#bab0ac"]


@dataclass
class Event:
    core_id: int
    cta_id: int
    kind: str  # mac | fixup_wait | fixup_reduce
    start: float
    end: float
    tile_idx: int


@dataclass
class Timeline:
    p: int
    events: List[Event]
    makespan: float


def from_device(records: np.ndarray) -> Timeline:
    """records: Gemm.timeline() rows [unit, tile, core, kind, t_mac_start, t_mac_end,
    t_wait_end, t_done].  `mac` covers the segment's mainloop; an owner with peers
    adds `fixup_wait` (until its peers' flags) and `fixup_reduce` (fold + store);
    every other segment's epilogue is folded into its `mac` event."""
    if len(records) == 0:
        return Timeline(1, [], 0.0)
    t0 = float(records[:, 4].min())
    us = lambda x: (float(x) - t0) * 1e-3  # noqa: E731
    events = []
    for u, tile, core, kind, ms, me, we, done in records.tolist():
        owner_with_peers = bool(kind & 2)
        events.append(Event(core, u, "mac", us(ms), us(me if owner_with_peers else done), tile))
        if owner_with_peers:
            events.append(Event(core, u, "fixup_wait", us(me), us(we), tile))
            events.append(Event(core, u, "fixup_reduce", us(we), us(done), tile))
    events.sort(key=lambda e: (e.core_id, e.start))
    p = int(records[:, 2].max()) + 1
    return Timeline(p, events, max(e.end for e in events))


def utilization(tl: Timeline) -> float:
    """simulate.cpp:71-80: sum of mac durations / (p * makespan)."""
    if tl.makespan <= 0:
        return 0.0
    return sum(e.end - e.start for e in tl.events if e.kind == "mac") / (tl.p * tl.makespan)


def _fmt(v: float) -> str:
    return "%.6g" % v


def write_timeline_csv(tl: Timeline, out) -> None:
    """simulate.cpp:162-168 format: core_id,cta_id,kind,start,end."""
    out.write("core_id,cta_id,kind,start,end\n")
    for e in tl.events:
        out.write(f"{e.core_id},{e.cta_id},{e.kind},{_fmt(e.start)},{_fmt(e.end)}\n")


def render_gantt(tl: Timeline, out) -> None:
    """SVG Gantt in the layout of simulate.cpp:105-154: one row per core, one
    rectangle per event colour-keyed by tile, fixup events hatched.  It keeps
    the reference's geometry, palette and labels on purpose (§8(f) row 4 asks
    for output in the reference's format); it is a reporting helper, off the
    GEMM hot path."""
    chart_w, row_h, gap, left, top = 720.0, 26.0, 6.0, 64.0, 16.0
    height = top + tl.p * (row_h + gap) + 32.0
    width = left + chart_w + 16.0
    scale = chart_w / tl.makespan if tl.makespan > 0 else 1.0
    w = out.write
    w(f'<svg xmlns="http://www.w3.org/2000/svg" version="1.1" width="{_fmt(width)}" '
      f'height="{_fmt(height)}">\n')
    w('  <defs>\n    <pattern id="hatch" width="6" height="6" patternTransform="rotate(45)"'
      ' patternUnits="userSpaceOnUse">\n      <line x1="0" y1="0" x2="0" y2="6" stroke="#444444"'
      ' stroke-width="2"/>\n    </pattern>\n  </defs>\n')
    for core in range(tl.p):
        y = top + core * (row_h + gap)
        w(f'  <text x="4" y="{_fmt(y + row_h * 0.7)}" font-family="monospace" font-size="12">'
          f'core {core}</text>\n')
        w(f'  <rect x="{_fmt(left)}" y="{_fmt(y)}" width="{_fmt(chart_w)}" height="{_fmt(row_h)}"'
          ' fill="#f2f2f2"/>\n')
    for e in tl.events:
        if e.end <= e.start:
            continue
        y = top + e.core_id * (row_h + gap)
        x, ww = left + e.start * scale, (e.end - e.start) * scale
        w(f'  <rect x="{_fmt(x)}" y="{_fmt(y)}" width="{_fmt(ww)}" height="{_fmt(row_h)}" '
          f'fill="{PALETTE[e.tile_idx % len(PALETTE)]}" stroke="#333333" stroke-width="0.5"/>\n')
        if e.kind != "mac":
            w(f'  <rect x="{_fmt(x)}" y="{_fmt(y)}" width="{_fmt(ww)}" height="{_fmt(row_h)}" '
              'fill="url(#hatch)"/>\n')
    ay = top + tl.p * (row_h + gap) + 8.0
    w(f'  <line x1="{_fmt(left)}" y1="{_fmt(ay)}" x2="{_fmt(left + chart_w)}" y2="{_fmt(ay)}" '
      'stroke="#000000" stroke-width="1"/>\n')
    w(f'  <text x="{_fmt(left)}" y="{_fmt(ay + 14.0)}" font-family="monospace" '
      'font-size="12">0</text>\n')
    w(f'  <text x="{_fmt(left + chart_w - 40.0)}" y="{_fmt(ay + 14.0)}" font-family="monospace" '
      f'font-size="12">{_fmt(tl.makespan)}</text>\n</svg>\n')
