"""SH-only refit (drop-in for splattint/optimize.py) on the device engine.

`adam_step` and `optimize_iteration` keep the reference's per-call contract
(host numpy in, host numpy out).  `BackgroundOptimizer` keeps all state in HBM
(`engine.RefitEngine`) and only crosses the PCIe bus for metrics (batched) and
for `current_scene()` / `snapshot()` materialisation.

Precision: SH, Adam moments and arithmetic are float32 on the device.  Host
scenes are updated by *delta* (sh64 + (new32 - old32)), so coefficients the
optimizer does not move stay bit-identical to the caller's float64 values
(fixed points, unselected gaussians).
"""

from __future__ import annotations

import ctypes
import logging
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as D
from .engine import RefitEngine
from .errors import ValidationError
from .losses import DEFAULT_LAMBDA, LossBreakdown
from .render import DEFAULT_CONFIG

log = logging.getLogger(__name__)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


@dataclass(frozen=True)
class OptimizerConfig:
    lr_dc: float = 0.0025
    lr_rest: float = 0.000125
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    lam: float = DEFAULT_LAMBDA
    snapshot_every: int = 10


DEFAULT_OPTIMIZER = OptimizerConfig()


@dataclass(frozen=True)
class AdamState:
    m: np.ndarray
    v: np.ndarray
    step: int

    @classmethod
    def fresh(cls, n_gaussians: int) -> "AdamState":
        shape = (n_gaussians, 16, 3)
        return cls(m=np.zeros(shape), v=np.zeros(shape), step=0)


@dataclass(frozen=True)
class IterationMetrics:
    iteration: int
    view_id: int
    generation: int
    loss: LossBreakdown

    def line(self) -> str:
        """iter,viewId,generation,l1,ssim,total (optimize.py:86-96)."""
        return (f"{self.iteration},{self.view_id},{self.generation},"
                f"{self.loss.l1:.8f},{self.loss.ssim:.8f},{self.loss.total:.8f}")


@dataclass(frozen=True)
class OptimizerStatus:
    iteration: int
    loss: float
    ips: float
    generation: int


def _delta_to_host(base64: np.ndarray, old32: torch.Tensor, new32: torch.Tensor) -> np.ndarray:
    d = (new32.double() - old32.double()).cpu().numpy()
    return base64 + d


def adam_step(params, grads, state: AdamState, config: OptimizerConfig = DEFAULT_OPTIMIZER):
    """One bias-corrected Adam update (optimize.py:59-83) on the device."""
    params = np.asarray(params, dtype=np.float64)
    grads = np.asarray(grads, dtype=np.float64)
    if params.shape != grads.shape or params.ndim != 3 or params.shape[1:] != (16, 3):
        raise ValidationError(
            f"params/grads must both be (N, 16, 3), got {params.shape} and {grads.shape}")
    if not np.all(np.isfinite(grads)):
        log.warning("non-finite gradient; Adam iteration %d rejected", state.step + 1)
        return params, state
    p32 = D.to_device(params)
    p_new = p32.clone()
    m = D.to_device(state.m)
    v = D.to_device(state.v)
    g = D.to_device(grads)
    step = torch.tensor([state.step], dtype=torch.int64, device=p32.device)
    cfg = D.adam_config(config)
    N.call("rcgs_adam_dense", N.ptr(p_new), N.ptr(m), N.ptr(v), N.ptr(g), params.shape[0],
           ctypes.byref(cfg), None, N.ptr(step), D.stream_ptr())
    return (_delta_to_host(params, p32, p_new),
            AdamState(m=m.double().cpu().numpy(), v=v.double().cpu().numpy(), step=state.step + 1))


def optimize_iteration(scene, dataset, rng: np.random.Generator, state: AdamState,
                       config: OptimizerConfig = DEFAULT_OPTIMIZER):
    """One SH refit step on a uniformly sampled view (optimize.py:99-120)."""
    if len(dataset) == 0:
        raise ValidationError("dataset has no views")
    pick = int(rng.integers(len(dataset)))
    target = dataset.views[pick]
    view = target.view
    ds = D.device_scene(scene)
    sh32 = D.sh_to_device(scene.sh)
    eng = RefitEngine(ds, sh32.clone(), [(view.intrinsics, view.pose)],
                      [D.to_device(target.image)], config, cache_views=False)
    eng.m.copy_(D.to_device(state.m))
    eng.v.copy_(D.to_device(state.v))
    if eng.tile_state is not None:
        eng.tile_state.fill_(1)  # Adam state from the caller: no tile may be skipped
    eng.step_dev.fill_(state.step)
    eng.step(picks=[0])
    (_, _, l1, ss, total, rejected), = eng.drain()
    loss = LossBreakdown(l1=l1, ssim=ss, total=total, lam=config.lam)
    metrics = IterationMetrics(iteration=state.step + 1, view_id=view.view_id,
                               generation=dataset.generation, loss=loss)
    if rejected:
        log.warning("non-finite gradient; Adam iteration %d rejected", state.step + 1)
        return scene, state, metrics
    new_sh = _delta_to_host(scene.sh, sh32, eng.sh)
    new_state = AdamState(m=eng.m.double().cpu().numpy(), v=eng.v.double().cpu().numpy(),
                          step=state.step + 1)
    return scene.with_sh(new_sh), new_state, metrics


class BackgroundOptimizer:
    """Pausable refit worker with snapshots and atomic dataset swaps (optimize.py:131-259).

    All optimizer state lives on the device.  `run_iterations` is the
    deterministic synchronous mode; `start/pause/resume/stop` run the same
    loop on a worker thread with its own CUDA stream.  `views_per_step` > 1 or a
    `group` (torch.distributed process group, one rank per GPU) enables the
    view-batched multi-GPU step (engine.py).
    """

    def __init__(self, scene, dataset, config: OptimizerConfig = DEFAULT_OPTIMIZER, seed: int = 0,
                 metrics_sink=None, *, group=None, cache_views: bool = True,
                 stream_targets: bool = False, raster=DEFAULT_CONFIG, prefetch: int = 0):
        self._config = config
        self._scene0 = scene
        self._metrics_sink = metrics_sink
        # _lock guards the published state (re-entrant: _flush publishes under it);
        # _flush_lock serialises metric drains (worker and save_state); _step_lock is
        # held by whoever is enqueueing a step, so save_state / load_state / swaps
        # see the engine at a step boundary
        self._lock = threading.RLock()
        self._flush_lock = threading.RLock()
        self._step_lock = threading.Lock()
        self._cache_lock = threading.Lock()  # materialised snapshot / current scene caches
        self._exec_stream = None  # the stream the steps run on (worker or caller)
        self._dataset = dataset
        self._stream_targets = stream_targets
        self._raster = raster
        self._ds = D.device_scene(scene)
        self._sh0 = D.sh_to_device(scene.sh)
        # prefetch > 0 (only with cache_views=False) builds upcoming views on a side
        # stream; the view indices are then drawn `prefetch` steps ahead, so a
        # dataset swap takes effect after the already-drawn steps.
        self._engine = RefitEngine(self._ds, self._sh0.clone(), self._cameras(dataset),
                                   self._targets(dataset), config, seed=seed,
                                   cache_views=cache_views, group=group, raster=raster,
                                   prefetch=prefetch)
        # Adam publishes the post-step SH of every snapshot_every-th step into the
        # engine's snapshot buffer, in stream order (optimize.py:221-222)
        self._engine.enable_snapshots(config.snapshot_every)
        self._pending_dataset = None
        self._accepted = 0
        self._sh_base = None  # fp64 host SH on the device, uploaded on the first save_ply
        self._snapshot_cache = (None, None)  # (published step count, Scene)
        self._current_cache = (None, None)   # (step count, Scene)
        self._status = OptimizerStatus(0, 0.0, 0.0, dataset.generation)
        self._run_event = threading.Event()
        self._run_event.set()
        self._stop_event = threading.Event()
        self._thread = None
        self._window_start = time.perf_counter()
        self._window_iters = 0
        self._last_loss = 0.0

    # -- dataset plumbing -------------------------------------------------------
    @staticmethod
    def _view_ids(dataset):
        ids = getattr(dataset, "_rcgs_view_ids", None)
        if ids is None:
            ids = tuple(ev.view.view_id for ev in dataset.views)
            try:  # cached on the (frozen) dataset object
                object.__setattr__(dataset, "_rcgs_view_ids", ids)
            except Exception:
                pass
        return ids

    @staticmethod
    def _cameras(dataset):
        return [(ev.view.intrinsics, ev.view.pose) for ev in dataset.views]

    def _targets(self, dataset):
        if self._stream_targets:
            return [torch.from_numpy(np.ascontiguousarray(ev.image, np.float32)).pin_memory()
                    for ev in dataset.views]
        return [D.to_device(ev.image) for ev in dataset.views]

    def _apply_pending_dataset(self):
        """Swap in the dataset passed to swap_dataset (the reference reads it at
        the start of the next iteration, optimize.py:211-214).  Steps the
        prefetcher drew ahead are discarded and redrawn, so the next step samples
        the new dataset from the RNG state after the last executed step and
        fits its targets."""
        with self._lock:
            ds, self._pending_dataset = self._pending_dataset, None
        if ds is None:
            return
        if len(ds) == 0:
            raise ValidationError("dataset has no views")
        self._engine.set_dataset(self._cameras(ds), self._targets(ds))
        with self._lock:
            self._dataset = ds

    # -- state shared with other threads ------------------------------------------
    def _read_device(self, sh_dev, step_dev):
        """Consistent copy of (SH, step count) at a step boundary: one copy each,
        enqueued on the stream the steps run on (Adam is the only writer and is a
        single kernel on that stream), then waited for."""
        stream = self._exec_stream or torch.cuda.current_stream()
        with self._step_lock, torch.cuda.stream(stream):  # no Adam enqueued between the two copies
            sh = sh_dev.clone()
            step = step_dev.clone()
            done = torch.cuda.Event()
            done.record(stream)
        done.synchronize()
        return sh, int(step.item())

    def _materialise(self, sh_dev, step_dev, cache_name):
        # lock order: _step_lock (in _read_device) is never taken under _lock
        sh, step = self._read_device(sh_dev, step_dev)
        with self._cache_lock:
            ver, sc = getattr(self, cache_name)
            if ver == step and sc is not None:
                return sc
            sc = self._scene0.with_sh(_delta_to_host(self._scene0.sh, self._sh0, sh))
            setattr(self, cache_name, (step, sc))
            return sc

    def snapshot(self):
        """The scene published after the last step whose count is a multiple of
        snapshot_every (optimize.py:164-166, 226-230)."""
        return self._materialise(self._engine.snapshot_sh, self._engine.snapshot_step, "_snapshot_cache")

    def current_scene(self):
        return self._materialise(self._engine.sh, self._engine.step_dev, "_current_cache")

    def save_ply(self, path) -> None:
        """Checkpoint of the current SH (session.py:328-333 saves current_scene()
        through scene_io.py:156): encoded on the device from the live fp32 SH and
        byte-identical to save_scene_ply(self.current_scene())."""
        from .scene_io import save_scene_ply_device

        sh, _ = self._read_device(self._engine.sh, self._engine.step_dev)
        with self._cache_lock:
            if self._sh_base is None:
                self._sh_base = torch.from_numpy(np.ascontiguousarray(self._scene0.sh)).to(self._sh0.device)
            save_scene_ply_device(self._scene0, sh, path, sh_base=(self._sh_base, self._sh0))

    def save_state(self, path) -> None:
        """Optimizer checkpoint for an exact resume (an extension; the reference
        restarts Adam per session, session.py:355-358): SH, Adam moments and step,
        the view-sampling RNG and the views already drawn ahead, the accepted-step
        count.  Pending metrics are delivered to the sink first."""
        import json
        if self._thread is not None and not self.paused:
            raise ValidationError("save_state needs a paused or synchronous optimizer")
        with self._step_lock:  # waits for a step the worker was enqueueing at pause()
            with self._exec_ctx():
                self._flush()
                st = self._engine.state_dict()
            with self._lock:
                meta = {"rng": st["rng"], "ahead": st["ahead"], "step": st["step"], "accepted": self._accepted,
                        "n": int(st["sh"].shape[0])}
        np.savez(path, sh=st["sh"], m=st["m"], v=st["v"], meta=np.array(json.dumps(meta)))

    def load_state(self, path) -> None:
        """Restore `save_state` into a fresh optimizer built on the same scene,
        dataset cameras, config and world size; the next iterations then equal
        the ones the saved optimizer would have run, bit for bit."""
        import json
        if self._thread is not None:
            raise ValidationError("load_state must precede start()")
        with np.load(path) as z:
            meta = json.loads(str(z["meta"]))
            st = {"sh": z["sh"], "m": z["m"], "v": z["v"], "step": meta["step"], "rng": meta["rng"],
                  "ahead": meta["ahead"]}
        with self._step_lock, self._lock, self._cache_lock:
            self._engine.load_state_dict(st)
            self._accepted = int(meta["accepted"])
            self._engine.publish_now()  # the published snapshot is the restored SH
            torch.cuda.current_stream().synchronize()
            self._snapshot_cache = (None, None)
            self._current_cache = (None, None)

    def status(self) -> OptimizerStatus:
        with self._lock:
            return self._status

    def swap_dataset(self, dataset) -> None:
        with self._lock:
            self._pending_dataset = dataset

    @property
    def dataset(self):
        with self._lock:
            return self._dataset

    # -- control --------------------------------------------------------------------
    def start(self) -> None:
        if self._thread is not None:
            return
        self._thread = threading.Thread(target=self._loop, name="sh-refit", daemon=True)
        self._thread.start()

    def pause(self) -> None:
        self._run_event.clear()

    def resume(self) -> None:
        self._run_event.set()

    @property
    def paused(self) -> bool:
        return not self._run_event.is_set()

    def stop(self) -> None:
        self._stop_event.set()
        self._run_event.set()
        if self._thread is not None:
            self._thread.join(timeout=30.0)
            self._thread = None
        self._engine.close()

    @property
    def stopped(self) -> bool:
        return self._stop_event.is_set()

    # -- the loop -----------------------------------------------------------------------
    def _exec_ctx(self):
        return torch.cuda.stream(self._exec_stream) if self._exec_stream is not None else _nullctx()

    def _step(self) -> None:
        with self._step_lock:
            self._apply_pending_dataset()
            with self._lock:
                # the step's generation and the dataset's view ids travel with its
                # metrics (drained later, possibly after a swap)
                tag = (self._dataset.generation, self._view_ids(self._dataset))
            self._engine.step(generation=tag)
        self._window_iters += 1
        if len(self._engine.pending) >= min(self._config.snapshot_every, self._engine.max_pending):
            # non-blocking: starts the metrics read-back of the pending steps and
            # delivers the ones already landed (every step's metrics still reach the
            # sink, in order, one flush later) -- a blocking flush here drained the
            # whole step pipeline every `snapshot_every` iterations.  The snapshot
            # itself is published by the step's own Adam on the device.
            self._flush(wait=False)

    def _flush(self, wait: bool = True) -> None:
        with self._flush_lock:
            recs = self._engine.drain(wait)
            lines = []
            for picks, (gen, ids), l1, ss, total, rejected in recs:
                it = self._accepted + 1
                if rejected:
                    log.warning("non-finite gradient; Adam iteration %d rejected", it)
                else:
                    self._accepted += 1
                self._last_loss = total
                vid = ids[picks[self._engine.rank]]
                lines.append(IterationMetrics(iteration=it, view_id=vid, generation=gen,
                                              loss=LossBreakdown(l1, ss, total, self._config.lam)))
                if not rejected and self._accepted % self._config.snapshot_every == 0:
                    self._publish_status()
            if self._metrics_sink is not None:
                for m in lines:
                    self._metrics_sink(m)

    def _publish_status(self) -> None:
        now = time.perf_counter()
        elapsed = max(now - self._window_start, 1e-9)
        with self._lock:
            self._status = OptimizerStatus(iteration=self._accepted, loss=self._last_loss,
                                           ips=self._window_iters / elapsed,
                                           generation=self._dataset.generation)
        self._window_start = now
        self._window_iters = 0

    def _publish(self) -> None:
        """Publish the current scene now (run_iterations' final publish)."""
        with self._lock:
            self._engine.publish_now()
        self._publish_status()

    def _loop(self) -> None:
        stream = torch.cuda.Stream()
        self._exec_stream = stream
        with torch.cuda.stream(stream):
            while not self._stop_event.is_set():
                if not self._run_event.wait(timeout=0.1):
                    self._flush()
                    continue
                if self._stop_event.is_set():
                    break
                try:
                    self._step()
                except Exception:
                    log.exception("optimizer iteration failed; pausing")
                    self._run_event.clear()
            self._flush()

    def run_iterations(self, count: int):
        """Deterministic synchronous mode; returns the final scene."""
        if self._thread is not None:
            raise ValidationError("run_iterations cannot be mixed with a started worker")
        self._exec_stream = torch.cuda.current_stream()
        for _ in range(count):
            self._step()
        self._flush()
        self._publish()
        return self.current_scene()

    @property
    def engine(self) -> RefitEngine:
        return self._engine
