"""GPU phase timing and the Fig. 2-style profile report.

Mirror of the reference profiler (/root/reference/pkg/src/softmax_kit/
profiler.py): same public names and report layout, but every interval is a
pair of CUDA events on the launching stream, in integer nanosecond "ticks"
(``TICKS_PER_SECOND`` = 1e9, as the reference's perf_counter_ns ticks).

* ``time_whole``  -- the fused softmax (the hot path), one event pair per rep.
* ``time_phases`` -- the unfused MaxSub / Exp / SumScale kernels of
  ``phases.variant_pipeline`` with an event pair per phase plus an outer
  WholeOp pair, so MaxSub + Exp + SumScale <= WholeOp holds by construction.

Inputs may be a ``Matrix2D`` (copied to the device once, untimed) or a CUDA
tensor.  Unlike the CPU reference (which reuses one buffer, cache-warm), the
GPU timers rotate through enough copies of the input/output pair to span
>= 3x the 126 MB L2, so small shapes are timed against HBM, not L2.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from statistics import median
from typing import Sequence

from .errors import ArgumentError
from .kernels import KernelVariant, LaneConfig, softmax_into
from .tensor import Matrix2D

TICKS_PER_SECOND = 1_000_000_000
TICKS_PER_MS = TICKS_PER_SECOND // 1000


class PhaseId(Enum):
    MAXSUB = "MaxSub"
    EXP = "Exp"
    SUMSCALE = "SumScale"
    WHOLEOP = "WholeOp"


@dataclass(frozen=True)
class Timer:
    resolution: int
    source: str


def default_timer() -> Timer:
    return Timer(resolution=TICKS_PER_SECOND, source="cudaEventElapsedTime (ns ticks)")


@dataclass(frozen=True)
class PhaseTimings:
    maxsub: int
    exp: int
    sumscale: int
    whole: int

    @property
    def phase_sum(self) -> int:
        return self.maxsub + self.exp + self.sumscale

    def __getitem__(self, phase: PhaseId) -> int:
        return {PhaseId.MAXSUB: self.maxsub, PhaseId.EXP: self.exp,
                PhaseId.SUMSCALE: self.sumscale, PhaseId.WHOLEOP: self.whole}[phase]


def _device_input(m):
    import torch

    if isinstance(m, Matrix2D):
        return torch.from_numpy(m.view2d).cuda()
    if isinstance(m, torch.Tensor) and m.is_cuda and m.dim() == 2:
        return m.contiguous()
    raise ArgumentError("expected a Matrix2D or a 2-D CUDA tensor")


def _rotation(x, with_out: bool = True):
    """Copies of (x, out) spanning >= 3x L2 (bounded to 16 pairs)."""
    import torch

    l2 = torch.cuda.get_device_properties(x.device).L2_cache_size
    per = x.numel() * 4 * (2 if with_out else 1)
    n = int(max(1, min(16, -(-3 * l2 // max(per, 1)))))
    xs = [x] + [x.clone() for _ in range(n - 1)]
    ys = [torch.empty_like(x) for _ in range(n)]
    return xs, ys


def _check_reps(reps: int, warmup: int) -> None:
    if reps < 1:
        raise ArgumentError(f"reps must be >= 1, got {reps}")
    if warmup < 0:
        raise ArgumentError(f"warmup must be >= 0, got {warmup}")


def _ticks(e0, e1) -> int:
    return int(round(e0.elapsed_time(e1) * 1e6))


def _hold_stream(n_launches: int) -> None:
    """Park the stream behind a device-side sleep while the host enqueues the
    timed launches, so each event pair brackets GPU time only (not the
    host's per-launch latency while the GPU sits idle)."""
    import torch

    torch.cuda._sleep(int(min(2e9, 2e5 + n_launches * 1.2e5)))  # ~60 us of cycles per launch


def time_whole(m, variant: KernelVariant, reps: int, warmup: int = 10,
               cfg: LaneConfig = LaneConfig()) -> list[int]:
    """Device ticks of the fused softmax, one event pair per rep."""
    import torch

    _check_reps(reps, warmup)
    xs, ys = _rotation(_device_input(m))
    n = len(xs)
    for i in range(warmup):
        softmax_into(xs[i % n], ys[i % n], variant, cfg, check_finite=False)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    _hold_stream(reps)
    for i, (a, b) in enumerate(ev):
        a.record()
        softmax_into(xs[i % n], ys[i % n], variant, cfg, check_finite=False)
        b.record()
    torch.cuda.synchronize()
    return [_ticks(a, b) for a, b in ev]


def time_phases(m, variant: KernelVariant, reps: int, warmup: int = 10,
                cfg: LaneConfig = LaneConfig()) -> list[PhaseTimings]:
    """Per-phase device ticks of the unfused pipeline (profiler.py:96-133)."""
    import torch

    from .phases import variant_pipeline

    _check_reps(reps, warmup)
    xs, ys = _rotation(_device_input(m))
    n = len(xs)
    rows, cols = xs[0].shape
    pipe = variant_pipeline(variant, rows, cols, cfg)
    for i in range(warmup):
        pipe.maxsub(xs[i % n], ys[i % n])
        pipe.exp(ys[i % n])
        pipe.sumscale(ys[i % n])
    torch.cuda.synchronize()
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(reps)]
    _hold_stream(3 * reps)
    for i, e in enumerate(marks):
        x, dst = xs[i % n], ys[i % n]
        e[0].record()
        e[1].record()
        pipe.maxsub(x, dst)
        e[2].record()
        e[3].record()
        pipe.exp(dst)
        e[4].record()
        e[5].record()
        pipe.sumscale(dst)
        e[6].record()
        e[7].record()
    torch.cuda.synchronize()
    return [PhaseTimings(_ticks(e[1], e[2]), _ticks(e[3], e[4]), _ticks(e[5], e[6]),
                         _ticks(e[0], e[7])) for e in marks]


def phase_ratio_summary(timings: Sequence[PhaseTimings]) -> dict[PhaseId, float]:
    """Median per-execution share of WholeOp for each phase."""
    if not timings:
        raise ArgumentError("need at least one timing sample")
    out = {p: median(t[p] / t.whole for t in timings)
           for p in (PhaseId.MAXSUB, PhaseId.EXP, PhaseId.SUMSCALE)}
    out[PhaseId.WHOLEOP] = 1.0
    return out


# ---------------------------------------------------------------- reports
@dataclass(frozen=True)
class EventStats:
    name: str
    calls: int
    total: float
    min: float
    max: float
    ave: float
    ratio: float


@dataclass(frozen=True)
class ProfileReport:
    events: tuple[EventStats, ...]


REPORT_HEADER = "------------------------->     Profiling Report     <-----------------------"
_COLS = ("Event", "Calls", "Total", "Min.", "Max.", "Ave.", "Ratio.")


def build_report(events: Sequence[tuple[str, Sequence[float]]]) -> ProfileReport:
    """Aggregate tick samples per event, sorted by total descending; Ratio is
    the share of the grand total of all events (profiler.py:198-223)."""
    if not events:
        raise ArgumentError("build_report requires at least one event")
    rows = []
    for name, samples in events:
        if len(samples) == 0:
            raise ArgumentError(f"event {name!r} has no samples")
        tot = float(sum(samples))
        rows.append((name, len(samples), tot, float(min(samples)), float(max(samples))))
    grand = sum(r[2] for r in rows)
    stats = sorted((EventStats(n, c, t, lo, hi, t / c, t / grand if grand > 0 else 0.0)
                    for n, c, t, lo, hi in rows), key=lambda e: e.total, reverse=True)
    return ProfileReport(events=tuple(stats))


def _ms(ticks: float) -> str:
    return f"{ticks / TICKS_PER_MS:.6g}"


def format_report(r: ProfileReport, place: str = "GPU") -> str:
    """Fixed-column text table in ms (Fig. 2 layout)."""
    w = max(len("Event"), *(len(e.name) for e in r.events)) + 2
    out = [REPORT_HEADER, "", f"Place: {place}", "Time unit: ms",
           "Sorted by total time in descending order in the same thread", "",
           f"{_COLS[0]:<{w}}{_COLS[1]:<9}{_COLS[2]:<10}{_COLS[3]:<10}{_COLS[4]:<10}"
           f"{_COLS[5]:<11}{_COLS[6]}"]
    for e in r.events:
        out.append(f"{e.name:<{w}}{e.calls:<9}{_ms(e.total):<10}{_ms(e.min):<10}"
                   f"{_ms(e.max):<10}{_ms(e.ave):<11}{e.ratio:.3f}")
    return "\n".join(out) + "\n"


def report_to_csv(r: ProfileReport) -> str:
    out = [",".join(_COLS)]
    out += [f"{e.name},{e.calls},{_ms(e.total)},{_ms(e.min)},{_ms(e.max)},{_ms(e.ave)},"
            f"{e.ratio:.3f}" for e in r.events]
    return "\n".join(out) + "\n"


def parse_report(text: str) -> ProfileReport:
    """Inverse of format_report (times back to ticks)."""
    lines = text.splitlines()
    try:
        start = next(i for i, ln in enumerate(lines) if ln.startswith("Event"))
    except StopIteration:
        raise ArgumentError("no column header found in report text") from None
    evs = []
    for ln in lines[start + 1:]:
        if not ln.strip():
            continue
        name, calls, total, lo, hi, ave, ratio = ln.split()
        evs.append(EventStats(name, int(calls), float(total) * TICKS_PER_MS,
                              float(lo) * TICKS_PER_MS, float(hi) * TICKS_PER_MS,
                              float(ave) * TICKS_PER_MS, float(ratio)))
    return ProfileReport(events=tuple(evs))
