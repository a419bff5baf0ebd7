"""Device-resident recolor refit engine (the hot loop of optimize.py:99-120, 252-259).

One optimizer step for a view batch:
    K1+K2 view preprocess/binning (or a cached View: geometry is frozen)
    -> K1 colour from the current SH -> K3 forward raster
    -> K5 loss + image gradient (fp64) -> K6 backward (per-gaussian acc)
    -> [multi-GPU: all-gather of the N x 3 acc vectors over NCCL]
    -> K7 fused gradient expansion + Adam (device step counter, reject flag).
Everything stays in HBM; the host only draws view indices from the reference's
RNG stream and reads metrics back in batches.

Multi-GPU: every rank holds a replica of the gaussians, the SH
and the Adam state, and all views' targets.  A step draws G = world_size views
(`rng.integers(V, size=G)`, the same stream as G sequential draws); rank r
back-propagates view picks[r] and the ranks exchange only their N x 3
per-gaussian channel sums (12 B/gaussian instead of the 192 B dense gradient);
each rank then expands sum_v basis_v (x) acc_v / G for all G views in a fixed
order, so every replica applies the bit-identical Adam update without a
floating-point all-reduce.
"""

from __future__ import annotations

import collections
import os
import ctypes
import threading
import time

import numpy as np
import torch

from . import _native as N
from . import device as D
from . import parallel
from .render import DEFAULT_CONFIG


def cameras_equal(a, b) -> bool:
    """Value equality of [(intrinsics, pose)] lists (poses hold numpy arrays, whose
    dataclass __eq__ would raise)."""
    if len(a) != len(b):
        return False
    for (ia, pa), (ib, pb) in zip(a, b):
        if (ia.fx, ia.fy, ia.cx, ia.cy, ia.width, ia.height) != (ib.fx, ib.fy, ib.cx, ib.cy, ib.width, ib.height):
            return False
        if not (np.array_equal(np.asarray(pa.rotation), np.asarray(pb.rotation))
                and np.array_equal(np.asarray(pa.translation), np.asarray(pb.translation))):
            return False
    return True


class ViewPrefetcher:
    """Builds the views of upcoming steps on side streams from worker threads.

    A view build (K1 + depth sort + K2) synchronises its stream twice to size
    its buffers; running it one or two steps ahead on its own stream and host
    thread (ctypes releases the GIL) overlaps those syncs and the build kernels
    with the current step's raster / loss / backward / Adam.  Every step still
    builds its own view from scratch; only the timing moves.

    `workers` threads (RCGS_PREFETCH_WORKERS, default 2) take jobs in turn, each
    on its own stream: a build's wall time (its two host syncs, and kernels that
    only run between the main stream's CTAs) is about one step, so one worker
    cannot stay ahead; two interleave.  The streams run at the main stream's
    (normal) priority: at the highest priority (the round-1 choice) the queued build
    kernels took every SM the recording raster released and the loss waited ~58 us
    per step behind them (`tools/stream_gaps.py`); at equal priority the main
    stream's kernels start first and the builds fill in (1084.5 vs 1072.9
    view-steps/s).  RCGS_PREFETCH_PRIORITY overrides.

    Used views come back through `retire`: the worker that built a view frees it
    on ITS stream after an event recorded on the consumer's stream.  Allocation
    and release of view memory then happen on one stream, so the stream-ordered
    pool reuses blocks without cross-stream dependencies and never grows in
    steady state.  Growing it (a driver-locked physical allocation) stalled both
    host threads for 30-800 ms when views were freed on the consumer stream instead.
    """

    def __init__(self, dscene, cameras, raster, device, profile=False, targets=None, depth=2, workers=None):
        self.dscene, self.cameras, self.raster, self.device = dscene, cameras, raster, device
        self.profile = profile
        # host-resident targets (streamed datasets): each upcoming step's target is
        # uploaded on the side stream into a small device ring (copy engine,
        # overlapping compute); a slot is rewritten only after the step that read it
        # has been retired (its event)
        self.targets = targets if targets is not None and any(not t.is_cuda for t in targets) else None
        self.ring = [None] * (depth + 4)
        self.ring_free = [None] * (depth + 4)
        self.copy_stream = None  # one copy stream per worker (below): uploads of two steps run concurrently
        self.gate_event = None   # optional main-stream event the next uploads wait for
        self.events = []  # (start, end) of each view build on its side stream
        self.host_build_ms = []
        self.host_wait_ms = []
        if workers is None:
            workers = int(os.environ.get("RCGS_PREFETCH_WORKERS", "2"))
        workers = max(1, int(workers))
        prio = os.environ.get("RCGS_PREFETCH_PRIORITY")
        prio = int(prio) if prio is not None else 0
        self.streams = [torch.cuda.Stream(device=device, priority=prio) for _ in range(workers)]
        # per-worker copy streams: with one, the ~25 MB target uploads (one per step,
        # ~21 GB/s from pinned host memory) were serialised at about the step rate
        nc = int(os.environ.get("RCGS_UPLOAD_STREAMS", str(workers)))
        self.copy_streams = ([torch.cuda.Stream(device=device) for _ in range(max(1, nc))]
                             if self.targets is not None else [])
        self.jobs = collections.deque()
        self.retired = [collections.deque() for _ in range(workers)]
        self.builder = {}  # id(view) -> index of the worker that built it
        self.ready = {}
        self.cv = threading.Condition()
        self.stop = False
        self.error = None
        self.threads = [threading.Thread(target=self._run, args=(w,), name=f"view-prefetch-{w}", daemon=True)
                        for w in range(workers)]
        for t in self.threads:
            t.start()

    def set_dataset(self, cameras, targets) -> None:
        """New cameras / targets for builds submitted from now on (no job may be
        in flight: the engine takes every prefetched step first)."""
        host = targets if targets is not None and any(not t.is_cuda for t in targets) else None
        with self.cv:
            self.cameras = cameras
            if host is not None and not self.copy_streams:
                self.copy_streams = [torch.cuda.Stream(device=self.device) for _ in range(len(self.streams))]
            self.targets = host

    def submit(self, key, index):
        with self.cv:
            self.jobs.append((key, index))
            self.cv.notify_all()

    def retire(self, view, key=None):
        """Hand a used view back; it is freed on its builder's stream once the
        current stream's work queued so far (which reads the view) has completed.
        `key` releases the step's target-ring slot at the same event."""
        ev = torch.cuda.Event()
        ev.record()
        with self.cv:
            w = self.builder.pop(id(view), 0)
            self.retired[w].append((view, ev))
            if key is not None and self.targets is not None:
                self.ring_free[key % len(self.ring)] = ev
            self.cv.notify_all()

    def _free_retired(self, w):
        with self.cv:
            items = list(self.retired[w])
            self.retired[w].clear()
        for view, ev in items:
            self.streams[w].wait_event(ev)
            view.close()

    def take(self, key):
        t0 = time.perf_counter()
        with self.cv:
            while key not in self.ready and self.error is None:
                self.cv.wait(timeout=1.0)
            if self.profile:
                self.host_wait_ms.append((time.perf_counter() - t0) * 1000.0)
            if self.error is not None:
                raise self.error
            return self.ready.pop(key)

    def _run(self, w):
        torch.cuda.set_device(self.device)
        stream = self.streams[w]
        with torch.cuda.stream(stream):
            while True:
                with self.cv:
                    while not self.jobs and not self.retired[w] and not self.stop:
                        self.cv.wait(timeout=1.0)
                    if self.stop:
                        return
                    job = self.jobs.popleft() if self.jobs else None
                if job is None:
                    self._free_retired(w)
                    continue
                key, index = job
                try:
                    with self.cv:
                        intr, pose = self.cameras[index]
                        targets = self.targets
                    tgt, copied = None, None
                    if targets is not None:
                        # the upload runs on its own stream, concurrently with the build
                        src = targets[index]
                        slot = key % len(self.ring)
                        with self.cv:
                            free = self.ring_free[slot]
                        cs = self.copy_streams[w % len(self.copy_streams)]
                        with torch.cuda.stream(cs):
                            if free is not None:
                                cs.wait_event(free)
                            gate = self.gate_event
                            if gate is not None:  # RCGS_UPLOAD_GATE: not under the loss
                                cs.wait_event(gate)
                            if self.ring[slot] is None or self.ring[slot].shape != src.shape:
                                self.ring[slot] = torch.empty(src.shape, dtype=torch.float32, device=self.device)
                            tgt = self.ring[slot]
                            tgt.copy_(src, non_blocking=True)
                            copied = torch.cuda.Event()
                            copied.record(cs)
                    t0 = time.perf_counter()
                    if self.profile:
                        e0 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                    if _BUILD_GATE and self.gate_event is not None:  # builds start after a backward
                        stream.wait_event(self.gate_event)
                    view = D.View(self.dscene, intr, pose, self.raster)
                    if self.profile:
                        self.host_build_ms.append((time.perf_counter() - t0) * 1000.0)
                    if copied is not None:
                        stream.wait_event(copied)  # one ready event covers view + target
                    ev = torch.cuda.Event(enable_timing=self.profile)
                    ev.record(stream)
                    if self.profile:
                        self.events.append((e0, ev))
                    with self.cv:
                        self.builder[id(view)] = w
                        self.ready[key] = (view, ev, tgt)
                        self.cv.notify_all()
                    self._free_retired(w)
                except Exception as e:  # surfaced to the consumer
                    with self.cv:
                        self.error = e
                        self.cv.notify_all()
                    return

    def close(self):
        with self.cv:
            self.stop = True
            self.cv.notify_all()
        for t in self.threads:
            t.join(timeout=30)
        for w, stream in enumerate(self.streams):
            with torch.cuda.stream(stream):
                self._free_retired(w)
        for view, _, _ in self.ready.values():
            w = self.builder.pop(id(view), 0)
            with torch.cuda.stream(self.streams[w]):
                view.close()
        self.ready.clear()


# Streamed targets: the next uploads wait for this step's backward ("bwd", default)
# or loss ("loss") on the optimizer stream, so the 25 MB DMA runs under Adam and the
# next raster instead of under the loss and the record stream (the loss's gradient
# maps live in L2 between its passes).  e2e: none 1039, loss 1051, bwd 1058
# view-steps/s ("none": no gate).
_UPLOAD_GATE = os.environ.get("RCGS_UPLOAD_GATE", "bwd")
# View builds likewise start after a backward on the optimizer stream (default on):
# the loss then runs with fewer concurrent build kernels (1110 / 1064 vs 1108 / 1057
# view-steps/s value / e2e).
_BUILD_GATE = os.environ.get("RCGS_BUILD_GATE", "1") == "1"


class RefitEngine:
    def __init__(self, dscene: D.DeviceScene, sh_dev: torch.Tensor, cameras, targets,
                 config, seed: int = 0, cache_views: bool = True, views=None, group=None,
                 raster=DEFAULT_CONFIG, max_pending: int = 4096, prefetch: int = 0,
                 profile: bool = False, fuse_color: bool = True, sparse_adam: bool = False):
        self.dscene = dscene
        self.sh = sh_dev                      # (N, 16, 3) fp32, updated in place
        self.m = torch.zeros_like(sh_dev)
        self.v = torch.zeros_like(sh_dev)
        # 64-gaussian tiles whose Adam state may be nonzero (exact skipping of
        # never-touched tiles, rcgs_adam_fused_ex); reset to ones by state loads
        # off by default: at C3 every 64-gaussian tile is touched within a few steps
        # (measured 99.8%), so the skip only pays for small edits
        sparse_adam = sparse_adam or os.environ.get("RCGS_SPARSE_ADAM", "0") == "1"
        self.tile_state = (torch.zeros((dscene.n + 63) // 64, dtype=torch.int32, device=sh_dev.device)
                           if sparse_adam else None)
        self.cameras = list(cameras)          # [(intrinsics, pose)]
        self.targets = targets                # per view (H, W, 3) fp32 device or pinned host
        self.config = config
        self.raster = raster
        self.rng = np.random.default_rng(seed)
        self.cache_views = cache_views
        self.views = views if views is not None else [None] * len(self.cameras)
        self.group = group
        self.world, self.rank = parallel.world_of(group)
        dev = D.device()
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self.reject = torch.zeros(1, dtype=torch.int32, device=dev)
        self.acc = torch.empty((dscene.n, 3), dtype=torch.float32, device=dev)
        self.acc_all = (torch.empty((self.world, dscene.n, 3), dtype=torch.float32, device=dev)
                        if self.world > 1 else None)
        self.max_pending = max_pending
        self.records = torch.zeros((max_pending, 4), dtype=torch.float64, device=dev)
        self.pending = []                     # [(picks, generation)]
        self._bufs = {}
        self._adam_cfg = D.adam_config(config)
        self._centers = [D.camera_center(pose) for _, pose in self.cameras]
        # prefetch > 0: draw picks `prefetch` steps ahead and build their views on a
        # side stream (only without view caching; see ViewPrefetcher)
        self.prefetch = prefetch if not cache_views else 0
        self._future = collections.deque()
        self._seq = 0
        if self.prefetch:
            # up to prefetch + 1 views alive at once, ~170 B per gaussian each plus
            # build temporaries: grow the pool once, outside any timed region
            N.call("rcgs_pool_reserve", int((self.prefetch + 2) * dscene.n * 400), D.stream_ptr())
        self._pf = (ViewPrefetcher(dscene, self.cameras, raster, dev, profile, targets=self.targets,
                                   depth=self.prefetch) if self.prefetch else None)
        self._d2h = collections.deque()  # in-flight metric read-backs (drain(wait=False))
        # profile: CUDA events around every stage of every step (negligible cost)
        self.profile = profile
        self._prof = []
        self._build_ev = []  # inline view builds (no prefetcher)
        # with prefetching, Adam also colours the next step's view (rcgs_adam_fused_next)
        self.fuse_color = fuse_color and os.environ.get("RCGS_FUSE_COLOR", "1") != "0"
        self._held = None
        self._undo = {}  # key -> how to undo the draw of a step taken ahead (reset_ahead)
        # snapshot publication inside Adam (enable_snapshots): the post-step SH of
        # every step whose count is a multiple of `every`, written in stream order
        self._publish = None
        self.snapshot_sh = None
        self.snapshot_step = None

    def enable_snapshots(self, every: int) -> None:
        """Have every Adam step whose committed count is a multiple of `every`
        also write the updated SH to `snapshot_sh` (and the count to
        `snapshot_step`) in stream order: the reference's publication of the
        post-step scene (optimize.py:221-222, 226-238) with no host round trip."""
        if every <= 0:
            raise ValueError("snapshot cadence must be positive")
        self.snapshot_sh = self.sh.clone()
        self.snapshot_step = self.step_dev.clone()
        self._publish = N.AdamPublish(self.snapshot_sh.data_ptr(), self.snapshot_step.data_ptr(), int(every))

    def publish_now(self) -> None:
        """Copy the current SH and step count into the snapshot (on the current stream)."""
        self.snapshot_sh.copy_(self.sh)
        self.snapshot_step.copy_(self.step_dev)

    def close(self):
        if self._held is not None:
            self._pf.retire(self._held[1])
            self._held = None
        if self._pf is not None:
            self._pf.close()
            while self._future:
                self._future.popleft()
            self._pf = None

    # -- helpers ------------------------------------------------------------------
    def view(self, i: int) -> D.View:
        if self.cache_views:
            if self.views[i] is None:
                intr, pose = self.cameras[i]
                self.views[i] = D.View(self.dscene, intr, pose, self.raster)
            return self.views[i]
        intr, pose = self.cameras[i]
        return D.View(self.dscene, intr, pose, self.raster)

    def _buf(self, h, w):
        key = (h, w)
        if key not in self._bufs:
            dev = D.device()
            self._bufs[key] = (torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                               torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                               torch.empty((h, w, 3), dtype=torch.float32, device=dev))
        return self._bufs[key]

    def draw(self):
        """View indices of the next step from the reference RNG stream (optimize.py:106)
        -- after any picks restored by `load_state` that were drawn before it."""
        return self._draw()[0]

    def _draw(self):
        """(picks, undo): undo restores the RNG / replay queue to before this draw."""
        replay = getattr(self, "_replay", None)
        if replay:
            return replay.popleft(), ("replay", None)
        state = self.rng.bit_generator.state
        return parallel.draw_views(self.rng, len(self.cameras), self.world), ("rng", state)

    def reset_ahead(self) -> None:
        """Discard the steps drawn ahead by the prefetcher (their views are built,
        not executed) and undo their draws, so the next step draws again from the
        RNG state after the last executed step.  Used by dataset swaps, which the
        reference applies from the next iteration on (optimize.py:173-175, 211-214)."""
        if self._pf is None:
            return
        taken = []
        if self._held is not None:
            picks, view, _, key, _ = self._held
            self._held = None
            self._pf.retire(view, key)
            taken.append((key, picks))
        while self._future:
            key, picks = self._future.popleft()
            view, ev, _ = self._pf.take(key)
            torch.cuda.current_stream().wait_event(ev)
            self._pf.retire(view, key)
            taken.append((key, picks))
        taken.sort()
        replayed = []
        first_rng = None
        for key, picks in taken:
            kind, state = self._undo.pop(key)
            if kind == "replay":
                replayed.append(list(picks))
            elif first_rng is None:
                first_rng = state
        if first_rng is not None:
            self.rng.bit_generator.state = first_rng
        if replayed:
            self._replay = collections.deque(replayed + list(getattr(self, "_replay", ())))

    def set_dataset(self, cameras, targets) -> None:
        """Swap the views' targets (and cameras, if they differ) from the next step on."""
        self.reset_ahead()
        cameras = list(cameras)
        if not cameras_equal(cameras, self.cameras):
            for v in self.views:
                if v is not None:
                    v.close()
            self.cameras = cameras
            self.views = [None] * len(cameras)
            self._centers = [D.camera_center(p) for _, p in cameras]
        self.targets = targets
        if self._pf is not None:
            self._pf.set_dataset(self.cameras, targets)

    # -- optimizer state (checkpoint / resume) -------------------------------------
    def state_dict(self) -> dict:
        """Exact resume state: SH / Adam moments / step counter, the RNG, and the
        picks already drawn for steps not yet executed (prefetch draws ahead).
        Pending metrics are not included; drain() first."""
        ahead = []
        if self._held is not None:
            ahead.append(list(self._held[0]))
        ahead += [list(p) for _, p in self._future]
        ahead += [list(p) for p in getattr(self, "_replay", ())]
        return {"sh": self.sh.cpu().numpy(), "m": self.m.cpu().numpy(), "v": self.v.cpu().numpy(),
                "step": int(self.step_dev.item()), "rng": self.rng.bit_generator.state, "ahead": ahead}

    def load_state_dict(self, st: dict) -> None:
        """Restore `state_dict()` into a fresh engine (same scene, views and world size)."""
        if self._held is not None or self._future:
            raise RuntimeError("load_state_dict needs an engine that has not stepped")
        for name in ("sh", "m", "v"):
            src = torch.as_tensor(np.ascontiguousarray(st[name], dtype=np.float32))
            dst = getattr(self, name)
            if tuple(src.shape) != tuple(dst.shape):
                raise ValueError(f"state {name} has shape {tuple(src.shape)}, engine {tuple(dst.shape)}")
            dst.copy_(src.to(dst.device))
        self.step_dev.fill_(int(st["step"]))
        if self.tile_state is not None:
            self.tile_state.fill_(1)  # m/v written from outside: every tile may be nonzero
        self.rng.bit_generator.state = st["rng"]
        self._replay = collections.deque([list(p) for p in st["ahead"]])
        torch.cuda.current_stream().synchronize()

    # -- one step -----------------------------------------------------------------
    def _next_prefetched(self):
        """(picks, view, coloured) of the next step: the view taken ahead (and
        coloured by the previous step's Adam epilogue) if any, else the next
        prefetched one."""
        if self._held is not None:
            held, self._held = self._held, None
            return held
        picks, view, key, tgt = self._take_prefetched()
        return picks, view, False, key, tgt

    def _take_prefetched(self):
        while len(self._future) < self.prefetch:
            picks, undo = self._draw()
            key = self._seq
            self._undo[key] = undo
            self._seq += 1
            self._pf.submit(key, picks[self.rank] if self.world > 1 else picks[0])
            self._future.append((key, picks))
        key, picks = self._future.popleft()
        view, ev, tgt = self._pf.take(key)
        torch.cuda.current_stream().wait_event(ev)
        return picks, view, key, tgt

    def step(self, picks=None, generation: int = 0):
        coloured = False
        key, tgt_pf = None, None
        if picks is None and self._pf is not None:
            picks, view, coloured, key, tgt_pf = self._next_prefetched()
            mine = picks[self.rank] if self.world > 1 else picks[0]
            prefetched = True
        else:
            prefetched = False
            picks = self.draw() if picks is None else picks
            mine = picks[self.rank] if self.world > 1 else picks[0]
            if self.profile:
                b0 = torch.cuda.Event(enable_timing=True)
                b0.record()
            view = self.view(mine)
            if self.profile:
                b1 = torch.cuda.Event(enable_timing=True)
                b1.record()
                self._build_ev.append((b0, b1))
        # stage events: colour | raster | loss | backward | (wait for the next view) | adam
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)] if self.profile else None
        if ev:
            ev[0].record()
        if not coloured:
            view.color(self.sh)
        img, tgt_buf, grad = self._buf(view.height, view.width)
        if ev:
            ev[1].record()
        view.render(None, 0, out=img, train=True)
        if self.cache_views:  # resident views also keep their weights (SpMV from then on)
            view.keep_records()
        target = self.targets[mine]
        if tgt_pf is not None:           # streamed dataset, uploaded by the prefetcher
            target = tgt_pf
        elif not target.is_cuda:         # streamed dataset: H2D of this step's target
            tgt_buf.copy_(target, non_blocking=True)
            target = tgt_buf
        slot = len(self.pending) % self.max_pending
        rec = self.records[slot]
        if ev:
            ev[2].record()
        D.loss_grad(img, target, self.config.lam, loss3=rec[:3], grad=grad)
        if _UPLOAD_GATE == "loss" and self._pf is not None and self._pf.targets is not None:
            gate = torch.cuda.Event()
            gate.record()
            self._pf.gate_event = gate
        # self.reject is 0 here: the previous step's Adam consumed and re-armed it
        if ev:
            ev[3].record()
        view.backward(grad, acc=self.acc, nonfinite=self.reject)
        if self._pf is not None and ((_UPLOAD_GATE == "bwd" and self._pf.targets is not None) or _BUILD_GATE):
            gate = torch.cuda.Event()
            gate.record()
            self._pf.gate_event = gate
        accs = parallel.exchange_accs(self.acc, self.group, out=self.acc_all)
        parallel.any_rank(self.reject, self.group)
        if ev:
            ev[4].record()
        ptrs = (ctypes.c_void_p * len(accs))(*[a.data_ptr() for a in accs])
        cen = np.concatenate([self._centers[p] for p in picks[:len(accs)]])
        args = (self.dscene.handle, N.ptr(self.sh), N.ptr(self.m), N.ptr(self.v), ptrs,
                (ctypes.c_double * len(cen))(*cen), len(accs), ctypes.byref(self._adam_cfg),
                N.ptr(self.reject), N.ptr(self.step_dev), N.ptr(rec[3:4]))
        pub = ctypes.byref(self._publish) if self._publish is not None else None
        if prefetched and self.fuse_color:
            # take the next step's view now (its build was submitted `prefetch`
            # steps ago; the stream waits for it before the Adam stage event) and
            # let this Adam colour it from the updated SH
            nxt_picks, nxt, nxt_key, nxt_tgt = self._take_prefetched()
            if ev:
                ev[5].record()
            # also records + re-arms the reject flag, and publishes snapshots
            N.call("rcgs_adam_fused_ex", *args, nxt.handle, pub, N.ptr(self.tile_state), D.stream_ptr())
            nxt._colored = True
            self._held = (nxt_picks, nxt, True, nxt_key, nxt_tgt)
        else:
            if ev:
                ev[5].record()
            N.call("rcgs_adam_fused_ex", *args, None, pub, N.ptr(self.tile_state), D.stream_ptr())
        if ev:
            ev[6].record()
            self._prof.append((ev, coloured))
        self.pending.append((picks, generation))
        if prefetched:
            self._undo.pop(key, None)
            self._pf.retire(view, key)
        elif not self.cache_views:
            view.close()
        return picks

    def drain(self, wait: bool = True):
        """Return [(picks, generation, l1, ssim, total, rejected)] of the steps whose
        metrics have reached the host.  wait=True synchronises on every pending
        step; wait=False starts a non-blocking read-back of the pending steps
        (pinned memory, stream ordered) and returns only those already landed --
        every step is still read back, one call later, without stalling the host
        pipeline."""
        if self.pending:
            n = len(self.pending)
            host = torch.empty((min(n, self.max_pending), 4), dtype=torch.float64, pin_memory=True)
            host.copy_(self.records[:host.shape[0]], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._d2h.append((ev, host, self.pending))
            self.pending = []
        out = []
        while self._d2h and (wait or self._d2h[0][0].query()):
            ev, host, pend = self._d2h.popleft()
            ev.synchronize()
            recs = host.numpy()
            for i, (picks, gen) in enumerate(pend):
                r = recs[i % self.max_pending]
                out.append((picks, gen, float(r[0]), float(r[1]), float(r[2]), bool(r[3] != 0)))
        return out

    def stage_report(self, reset: bool = True) -> dict:
        """Mean device ms per stage over the profiled steps (CUDA events on the
        launching streams; view builds on the prefetch stream)."""
        torch.cuda.synchronize()
        names = ["color", "raster_fwd", "loss_grad", "raster_bwd", "next_view_wait", "adam"]
        out = {}
        if self._prof:
            for i, nme in enumerate(names):
                # colour: only steps that launched the colour kernel (else it was
                # fused into the previous step's Adam, which the adam stage includes)
                ts = [e[i].elapsed_time(e[i + 1]) for e, fused in self._prof if not (i == 0 and fused)]
                if ts:
                    out[nme] = float(np.mean(ts))
            out["step_events"] = len(self._prof)
            out["color_fused_steps"] = sum(1 for _, fused in self._prof if fused)
        if self._pf is not None and self._pf.events:
            out["view_build"] = float(np.mean([a.elapsed_time(b) for a, b in self._pf.events]))
            if self._pf.host_build_ms:
                out["prefetch_host_build_ms_max"] = float(np.max(self._pf.host_build_ms))
                out["prefetch_wait_ms_max"] = float(np.max(self._pf.host_wait_ms or [0.0]))
        elif self._build_ev:
            out["view_build"] = float(np.mean([a.elapsed_time(b) for a, b in self._build_ev]))
        if reset:
            self._prof = []
            self._build_ev = []
            if self._pf is not None:
                self._pf.events = []
                self._pf.host_build_ms = []
                self._pf.host_wait_ms = []
        return out

    def step_count(self) -> int:
        return int(self.step_dev.item())
