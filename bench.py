#!/usr/bin/env python
"""Benchmark: deep-copy + leaf-kernel effective GB/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the hot path over one synthetic object graph:
  * value  -- the graph already resident in HBM: relocation (attach) -> pointerchain resolve ->
              leaf kernel -> detach, graph bytes / device time (CUDA events, max over ranks);
  * e2e    -- the same through the C-ABI window from pinned HOST buffers: chunked multi-stream
              H2D + relocation tables, the device work, and the D2H copy-back of the whole arena
              inside the timed region (harness.py:369-373 metered window).
Default workload C2: DenseSpec(q=4, depth=3, n=4Mi) float32 leaves-only -- a depth-4 pointer
chain (3 Lnext hops + A) to each of 64 leaf arrays of 4Mi floats, 1 GiB of payload.
Under torchrun each rank (one GPU) processes its own C2-shaped subtree shard: weak scaling,
no collective on the data path (gloo only for the barrier and the max-over-ranks timing).
``--impl reference`` times the CPU restatement of the reference path (oracle/, all host cores)
on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "deep-copy+kernel effective GB/s (H2D and HBM % of roofline) at 1/2/4/8 B200"

CONFIGS = {
    # name: (kind, args, elem, leaf_only, policy, description)
    "C1": ("linear", (1, 1_000_000, "allinit_allused"), 4, False, "all_arrays",
           "C1: depth-1 struct with one float32 leaf array of 1M elements"),
    "C2": ("dense", (4, 4 << 20, 3), 4, True, "all_leaves",
           "C2: depth-4 pointer chain, dense q=4 layout, 64 leaf arrays x 4Mi float32 (leaves only)"),
    "C3": ("forest", (4, 4 << 20, "LLinit_LLused"), 4, False, "all_leaves",
           "C3: 64 x depth-4 linear chains (LLinit_LLused), 64 leaves x 4Mi float32, 320 objects scattered "
           "over the slab (seeded permutation)"),
    "C4": ("dense", (100, 256, 3), 4, False, "all_leaves",
           "C4: 1,010,101 structs, 1M leaves x 256 float32, depth 3, relocation-bound"),
    "C5": ("dense", (4, 268_435_456, 3), 4, True, "all_leaves",
           "C5: 64 GiB depth-4 dense graph (64 leaves x 256Mi float32) per shard"),
}


def make_spec(name: str):
    from paper_1906_01128_b200 import DenseSpec, ForestSpec, LinearSpec
    kind, args, elem, leaf_only, policy, desc = CONFIGS[name]
    if kind == "forest":
        return ForestSpec(LinearSpec(*args, elem=elem), 64, scatter_seed=0xC3), policy, desc
    if kind == "linear":
        return LinearSpec(*args, elem=elem), policy, desc
    return DenseSpec(*args, elem=elem, leaf_only=leaf_only), policy, desc


# ------------------------------------------------------------------------------ distributed
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and clock-event reasons through NVML while the timed regions run."""

    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
               "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device: int, period_s: float = 0.05):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.period = period_s

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.nv:
            self._thr = threading.Thread(target=self._loop, daemon=True)
            self._thr.start()

    def stop(self) -> dict:
        if self._thr:
            self._stop.set()
            self._thr.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def measured_peaks() -> dict:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "MEASURED_PEAKS.json (measured)"}
    return {"hbm_gbs": 6650.0, "source": "B200_PROFILING.md fallback"}


def ncu_record(config: str) -> dict:
    """k_scale's `ncu --set full` numbers for this config (profiles/ncu_traffic.json), if captured."""
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        return json.loads(p.read_text()).get(config, {}).get("k_scale") or {}
    return {}


def ncu_traffic(config: str):
    return ncu_record(config).get("dram_bytes_per_launch")


# nominal B200 HBM3e bandwidth (vendor figure), reported beside the measured-copy roofline
NOMINAL_HBM_GBS = 8000.0


# ------------------------------------------------------------------------------ CPU legs
CPU_SAMPLE_BYTES = 2 << 30  # bound on the CPU leg's working set (3 buffers of this size)


def cpu_sample_spec(spec):
    """The CPU legs run the same tree shape; leaves are shortened so one graph <= 2 GiB."""
    from dataclasses import replace
    from paper_1906_01128_b200.scenarios import tree_total_bytes
    total = tree_total_bytes(spec, 16)
    if total <= CPU_SAMPLE_BYTES:
        return spec, 1
    f = -(-total // CPU_SAMPLE_BYTES)
    return replace(spec, n=spec.n // f), f


def cpu_window(spec, policy: str, seed: int, steps: int, warmup: int, threads: int):
    """The oracle's restatement of the metered window (host cores): copy in, attach, resolve,
    scale, detach, copy out.  Returns (seconds per step list, graph bytes)."""
    from oracle import oracle as O
    trees = 1
    if spec.__class__.__name__ == "ForestSpec":   # the reference has no forest: one tree x count
        spec, trees = spec.tree, spec.count
    ospec = O.OSpec(O.DENSE if spec.__class__.__name__ == "DenseSpec" else O.LINEAR,
                    getattr(spec, "q", getattr(spec, "k", 1)), spec.n, getattr(spec, "depth", 0),
                    getattr(spec, "layout", "allinit_allused"), spec.elem, getattr(spec, "leaf_only", False), 16)
    t = O.build(ospec, seed)
    pol = {"ref": O.TARGET_REF, "all_leaves": O.TARGET_ALL_LEAVES, "all_arrays": O.TARGET_ALL_ARRAYS}[policy]
    idx = O.targets(t, pol)
    keys = O.chain_keys(t, idx)
    dev = np.empty_like(t.buf)
    out = np.empty_like(t.buf)
    dev_base = 0x7E00_0000_0000
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        rc = O.window(t, idx, dev, out, t.ptr_base, dev_base, 2.0 if i % 2 == 0 else 0.5, threads, keys=keys)
        dt = time.perf_counter() - t0
        if rc != -1:
            raise RuntimeError(f"oracle window reported site {rc}")
        if i >= warmup:
            times.append(dt)
    return [x * trees for x in times], t.total * trees


def compare_schemes(spec, policy: str, reps: int, device: int) -> dict:
    """The four transfer schemes of the reference (harness.py:219-325) through the drop-in API on
    the same graph: window = transfer_to_device -> kernel_scale -> copy_back, host wall clock
    with device syncs, median of `reps` after one warm-up.  UVM is measured without hints and
    with a whole-tree prefetch; GB/s are graph bytes over the window."""
    import paper_1906_01128_b200 as cf
    out = {}
    plans = (("marshalling", "marshalling", {}), ("marshalling_eager", "marshalling", {"fused": False}),
             ("pointerchain", "pointerchain", {}), ("naive", "naive", {}),
             ("uvm", "uvm", {"uvm_hints": "none"}), ("uvm_prefetch", "uvm", {"uvm_hints": "prefetch"}),
             ("uvm_advise", "uvm", {"uvm_hints": "advise"}), ("uvm_preferred", "uvm", {"uvm_hints": "preferred"}),
             ("uvm_read_mostly", "uvm", {"uvm_hints": "read_mostly"}))
    for name, scheme, kw in plans:
        m = cf.Machine(device=device)
        try:
            if scheme == "uvm":
                m.enable_uvm()
            if scheme == "marshalling":
                arena, h = cf.marshal_tree(m, spec, seed=1, align=16)
            else:
                arena, h = None, cf.build_tree(m, spec, seed=1, align=16)
            times, h2d = [], 0
            for r in range(reps + 1):
                if r >= 2 and sum(times) > 30.0:   # keep the default run within minutes
                    break
                m.ctx.sync()
                mark = m.log.mark()
                t0 = time.perf_counter()
                prep = cf.transfer_to_device(m, h, scheme, arena, policy=policy, **kw)
                cf.kernel_scale(m, h, prep, 2.0 if r % 2 == 0 else 0.5)
                cf.copy_back(m, h, prep)
                m.ctx.sync()
                if r:
                    times.append(time.perf_counter() - t0)
                    h2d = m.log.bytes_moved("H2D", mark)
            med = statistics.median(times)
            out[name] = {"window_ms": round(med * 1e3, 3), "graph_gbs": round(h.total_bytes / med / 1e9, 3),
                         "h2d_bytes": int(h2d)}
        except Exception as exc:  # a scheme failing must not hide the others; it is reported
            out[name] = {"error": f"{type(exc).__name__}: {exc}"[:200]}
        finally:
            m.close()
    if "uvm" in out and "window_ms" in out["uvm"]:
        for v in out.values():
            if "window_ms" in v:
                v["normalized_to_uvm"] = round(v["window_ms"] / out["uvm"]["window_ms"], 4)
    return out


def run_reference(args, dist: Dist) -> None:
    if dist.rank != 0:
        return
    spec, policy, desc = make_spec(args.config)
    spec, shrink = cpu_sample_spec(spec)
    from oracle import oracle as O
    threads = O.default_threads()
    times, total = cpu_window(spec, policy, 1, args.steps, args.warmup, threads)
    per = statistics.fmean(times)
    gbs = total / per / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(per * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if args.config == "C5" else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (payload_values, seed 1)",
        "config": {"workload": desc, "graph_bytes": total, "parallelism": "host cores"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"full {args.config} window per step (oracle/cf_oracle.c, OpenMP)"
                                   + (f", leaves shortened {shrink}x to fit host RAM" if shrink > 1 else "")},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def verify_gather(w, shard, spec, dist: Dist, device: int, ndev: int, src_factor: float) -> dict:
    """Outside the timed region: one more window (scale 2.0) from the host arena, per-leaf
    checksums of the device image (cf_checksum_ranges), all-gathered to every rank -- over NCCL
    when each rank has its own GPU, else gloo -- and checked on rank 0 against the checksums of
    the whole workload (payload_values * factor, the same for every leaf of a level)."""
    import numpy as np
    from paper_1906_01128_b200 import _native as N
    from paper_1906_01128_b200.shard import expected_checksum, gather_checksums, leaf_checksums
    st = w.run(scale=2.0)
    if st.bad != N.NO_BAD:
        raise SystemExit("verification window reported a device error")
    off, cnt = w.plan.table(N.CF_TAB_ARR_OFF), w.plan.table(N.CF_TAB_ARR_COUNT)
    lvl, od = w.plan.table(N.CF_TAB_ARR_LEVEL), w.plan.table(N.CF_TAB_ARR_ORDINAL)
    tg = w.targets
    sums = leaf_checksums(w.ctx, w.image, off[tg], cnt[tg], spec.elem)
    if len(set(lvl[tg].tolist())) != 1 or len(set(cnt[tg].tolist())) != 1:
        raise SystemExit("verify_gather expects targets of one level and length")
    nleaf_tree = int(len(tg)) if shard.scaling == "weak" else 0
    # weak: (rank, position) -- every rank owns a whole tree; strong: the global leaf ordinal
    keys = (np.arange(len(tg), dtype=np.int64) + np.int64(dist.rank) * (1 << 32)) if shard.scaling == "weak" \
        else od[tg].astype(np.int64)
    pg, dev, backend, err = None, None, "local", None
    if dist.world > 1:
        import torch
        import torch.distributed as tdist
        backend = "gloo"
        if ndev >= dist.world:   # one GPU per rank: the gather runs over NCCL (NVLink / NVSwitch)
            try:
                torch.cuda.set_device(device)
                pg, dev, backend = tdist.new_group(backend="nccl"), torch.device("cuda", device), "nccl"
                o, v = gather_checksums(keys, sums, pg, dev)
            except Exception as exc:   # keep the bench line; fall back to the gloo group
                err = f"{type(exc).__name__}: {exc}"[:200]
                pg, dev, backend = None, None, "gloo"
    if backend != "nccl":
        o, v = gather_checksums(keys, sums, pg, dev)
    out = {"backend": backend, "leaves": int(len(o)), "what": "per-leaf u32-word checksums after a "
           "verification window (scale 2.0), gathered to all ranks"}
    if err:
        out["nccl_error"] = err
    if dist.rank == 0:
        f = 2.0 * src_factor
        ok = True
        seeds = {}
        for key, val in zip(o.tolist(), v.tolist()):
            seed = shard.seed + (key >> 32) if shard.scaling == "weak" else shard.seed
            lv = int(lvl[tg[0]])
            if (seed, lv) not in seeds:
                seeds[(seed, lv)] = expected_checksum(seed, lv, int(cnt[tg[0]]), spec.elem, f)
            ok &= int(val) == seeds[(seed, lv)]
        want = (dist.world * nleaf_tree) if shard.scaling == "weak" else int(spec.q ** spec.depth)
        out["complete"] = int(len(o)) == want and len(set(o.tolist())) == len(o)
        out["checksums_match"] = bool(ok)
        if not (ok and out["complete"]):
            raise SystemExit(f"gathered result check failed: {out}")
    return out


# working sets below this are L2-flushed before every timed step (B200 L2 = 126 MB)
L2_FLUSH_BELOW = 512 << 20


class L2Flush:
    """Evicts the L2 between timed steps (a 512 MiB device memset on the context's compute stream,
    outside the timed region) and times each step on the device (CUDA events inside the window)."""

    def __init__(self, w):
        import ctypes as C
        from paper_1906_01128_b200 import _native as N
        self.N, self.w = N, w
        self.buf = C.c_void_p()
        N.check(N.lib().cf_dev_alloc(w.ctx.handle, L2_FLUSH_BELOW, C.byref(self.buf)))

    def flush(self) -> None:
        self.N.check(self.N.lib().cf_memset(self.w.ctx.handle, self.buf, 0x5A, L2_FLUSH_BELOW))

    def steps(self, flags: int, warmup: int, steps: int, dist):
        """warmup then steps windows in one batch, the L2 flushed before each (outside the timed
        intervals); stats.ms_total = the sum of the windows' own device intervals."""
        self.w.run_n_flushed(warmup, self.buf.value, L2_FLUSH_BELOW, flags=flags)
        dist.barrier()
        st = self.w.run_n_flushed(steps, self.buf.value, L2_FLUSH_BELOW, flags=flags)
        dist.barrier()
        return st

    def close(self) -> None:
        self.N.lib().cf_dev_free(self.w.ctx.handle, self.buf)


# ------------------------------------------------------------------------------ our arm
def run_ours(args, dist: Dist) -> None:
    from paper_1906_01128_b200 import DeepCopyWindow
    from paper_1906_01128_b200 import _native as N

    from paper_1906_01128_b200.shard import shard_for

    from paper_1906_01128_b200 import _native as Nn
    ndev = Nn.device_count()
    # one rank per GPU; ranks beyond the visible GPUs share them (plumbing runs on small boxes)
    device = dist.local_rank % max(ndev, 1)
    spec, policy, desc = make_spec(args.config)
    n_full = spec.tree.n if hasattr(spec, "tree") else spec.n
    if args.leaf_elems and args.leaf_elems < n_full:   # plumbing runs only: the same shape, shorter leaves
        from dataclasses import replace
        spec = replace(spec, tree=replace(spec.tree, n=args.leaf_elems)) if hasattr(spec, "tree") else \
            replace(spec, n=args.leaf_elems)
        desc += f" [leaves shortened to {args.leaf_elems} elements: plumbing run, not a bench value]"
    scaling = "strong" if args.config == "C5" else "weak"
    shard = shard_for(spec, dist.rank, dist.world, scaling)
    spec = shard.spec
    # pinned arenas next to this GPU's host link (multi-socket boxes)
    numa_node = Nn.gpu_numa_node(device) if ndev else -1
    t_build = time.perf_counter()
    w = DeepCopyWindow(spec, seed=shard.seed, policy=policy, mode="resolved", align=16, numa_node=numa_node,
                       chunk_bytes=args.chunk_mb << 20, device=device,
                       separate_output=spec.n * spec.elem * 64 <= (16 << 30))
    t_build = time.perf_counter() - t_build
    total = w.total
    # small graphs (C1: 4 MB): two steps of at least 1 MiB, so copy-out of the first half overlaps
    # copy-in of the second (measured: 0.173 -> 0.156 ms per C1 window; 8 x 512 KiB steps lose)
    if total <= 4 * w.chunk_bytes:
        w.chunk_bytes = min(w.chunk_bytes, max(1 << 20, ((total + 1) // 2 + (1 << 20) - 1) >> 20 << 20))
    leaf_bytes = int(sum(int(w.plan.table(N.CF_TAB_ARR_COUNT)[i]) for i in w.targets)) * spec.elem
    kernel_traffic = 2 * leaf_bytes  # read + write of every targeted element

    # host-link ceilings for this transfer pattern (copy-only windows, same chunks/streams)
    # double-buffered: two windows over the same arena, own images / copy-back buffers, so
    # step r+1 copies in while step r copies out (skipped when two images would not fit)
    twin = w.twin() if (w.dst != w.src and not args.single_buffer) else None
    link = {}
    for name, fl in (("h2d", N.CF_WIN_H2D), ("d2h", N.CF_WIN_D2H), ("bidir", N.CF_WIN_H2D | N.CF_WIN_D2H)):
        probe = (lambda n: w.run_pair_n(twin, n, flags=fl)) if twin else (lambda n: w.run_n(n, flags=fl))
        probe(2)
        st = probe(4)
        link[name] = (st.h2d_bytes + st.d2h_bytes) / (st.ms_total * 1e-3) / 1e9

    clocks = ClockSampler(device)
    clocks.start()
    # ---- e2e: host buffers in, copy-back out, through the C-ABI window
    gflag = 0 if args.no_graph else N.CF_WIN_GRAPH
    run_e2e = (lambda n: w.run_pair_n(twin, n, flags=N.CF_WIN_FULL | gflag)) if twin else \
        (lambda n: w.run_n(n, flags=N.CF_WIN_FULL | gflag))
    flush = L2Flush(w) if total < L2_FLUSH_BELOW else None
    if flush is None:
        run_e2e(args.warmup)
        dist.barrier()
        N.check(N.lib().cf_ctx_sync(w.ctx.handle))
        st_e2e = run_e2e(args.steps)
        N.check(N.lib().cf_ctx_sync(w.ctx.handle))
        dist.barrier()
    else:   # working set fits L2: flush it before every step, time each step on the device
        st_e2e = flush.steps(N.CF_WIN_FULL | gflag, args.warmup, args.steps, dist)
    e2e_ms = dist.max(st_e2e.ms_total) / args.steps
    # ---- value: image resident in HBM
    w.upload_raw()
    if flush is None:
        w.run_n(args.warmup, flags=N.CF_WIN_RESIDENT | gflag)
        dist.barrier()
        N.check(N.lib().cf_ctx_sync(w.ctx.handle))
        st_res = w.run_n(args.steps, flags=N.CF_WIN_RESIDENT | gflag)
        N.check(N.lib().cf_ctx_sync(w.ctx.handle))
        dist.barrier()
    else:
        st_res = flush.steps(N.CF_WIN_RESIDENT | gflag, args.warmup, args.steps, dist)
    res_ms = dist.max(st_res.ms_total) / args.steps
    # ---- leaf-kernel duration (events around the k_scale launch, resident, after warm-up)
    kms = []
    for i in range(max(5, args.steps // 2)):
        if flush is not None:
            flush.flush()
        s = w.run_resident(scale=2.0 if i % 2 == 0 else 0.5)
        kms.append(s.ms_kernel)
    kernel_ms = statistics.fmean(kms)
    # ---- chase-per-access comparison (same resident image)
    chase = {}
    if not args.skip_chase:
        w.run_resident(scale=2.0, mode="chase")
        ck = [w.run_resident(scale=0.5 if i % 2 == 0 else 2.0, mode="chase") for i in range(4)]
        c_ms = statistics.fmean(s.ms_kernel for s in ck)
        chase = {"kernel_ms": round(c_ms, 4), "hbm_gbs": round(kernel_traffic / (c_ms * 1e-3) / 1e9, 1),
                 "resident_ms_per_step": round(statistics.fmean(s.ms_total for s in ck), 4)}
    clk = clocks.stop()

    # correctness spot check of the copy-back on the first and last targeted leaf
    arr = w.plan.table(N.CF_TAB_ARR_OFF)
    cnt = w.plan.table(N.CF_TAB_ARR_COUNT)
    lvl = w.plan.table(N.CF_TAB_ARR_LEVEL)
    dt = np.float32 if spec.elem == 4 else np.float64
    last = twin if (twin is not None and flush is None and (args.steps - 1) % 2 == 1) else w
    if w.dst != w.src:
        factor = 2.0 if (args.steps - 1) % 2 == 0 else 0.5      # last run's scale, source untouched
    else:
        factor = 2.0 ** (args.warmup % 2 + args.steps % 2)        # run_n alternates 2.0 / 0.5
    from paper_1906_01128_b200.scenarios import payload_values
    for i in (w.targets[0], w.targets[-1]):
        a, n_el = int(arr[i]), min(int(cnt[i]), 1 << 20)
        got = last.host_dst()[a:a + n_el * spec.elem].view(dt)
        want = (payload_values(shard.seed, int(lvl[i]), n_el, spec.elem) * dt(factor)).astype(dt)
        if not np.array_equal(got, want):
            raise SystemExit("copy-back spot check failed")

    gather = verify_gather(w, shard, spec, dist, device, ndev, 1.0 if w.dst != w.src else factor)

    n = dist.world
    graph_all = dist.sum(float(total))
    value = graph_all / (res_ms * 1e-3) / 1e9
    e2e = graph_all / (e2e_ms * 1e-3) / 1e9
    peaks = measured_peaks()
    achieved = kernel_traffic / (kernel_ms * 1e-3) / 1e9
    h2d_step = st_e2e.h2d_bytes // args.steps
    d2h_step = st_e2e.d2h_bytes // args.steps
    ideal_ms = (h2d_step + d2h_step) / (link["bidir"] * 1e9) * 1e3
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(res_ms, 4), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32" if spec.elem == 4 else "f64",
        "data": "synthetic (payload_values of the reference, seed 1+rank)",
        "config": {"workload": desc, "graph_bytes_per_gpu": total, "leaf_bytes_per_gpu": leaf_bytes,
                   "layout": "aligned16 arena", "targets": policy, "chunk_bytes": w.chunk_bytes,
                   "h2d_streams": 1, "d2h_streams": 1, "cuda_graph": not args.no_graph, "l2": "inputs >= 1 GiB per GPU exceed the 126 MB L2 (no flush needed)"
                   if flush is None else "working set below 512 MiB: L2 flushed (512 MiB device memset on the window's stream) "
                   "before every timed window, outside the timed intervals; per-window device intervals summed",
                   "parallelism": f"dp{n} ({scaling}-scaled subtree shards, one per GPU, no data-path collective)"},
        "e2e": {"value": round(e2e, 3), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": int(h2d_step), "d2h_bytes_per_step": int(d2h_step),
                "host_link_gbs": {k: round(v, 2) for k, v in link.items()},
                "host_link_probe": "copy-only windows, same chunking and buffering as the timed e2e",
                "ideal_ms_at_measured_bidir": round(ideal_ms, 3),
                "frac_of_link_roofline": round(ideal_ms / e2e_ms, 4),
                "gpu_launches_per_step": int(st_e2e.launches // args.steps),
                "double_buffered": twin is not None and flush is None},
        "roofline": {"bound": "hbm", "kernel": "k_scale<float,resolved>", "achieved": round(achieved, 1),
                     "peak": peaks["hbm_gbs"], "peak_source": peaks["source"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": ncu_traffic(args.config),
                     "frac_of_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                     "ncu_dram_pct_of_peak": ncu_record(args.config).get("dram_pct_of_ncu_peak"),
                     "algorithmic_bytes_per_launch": kernel_traffic, "kernel_ms": round(kernel_ms, 4),
                     "share_of_resident_step": round(kernel_ms / res_ms, 4)},
        "modes": {"resolved": {"kernel_ms": round(kernel_ms, 4), "hbm_gbs": round(achieved, 1)}, "chase": chase},
        "gpu_launches": int(st_res.launches),
        "numa": {"gpu_node": numa_node, "host_arenas": "allocated on the GPU's node" if numa_node >= 0 else "OS placement"},
        "gather": gather,
        "clocks": clk,
        "build_s": round(t_build, 2),
    }
    if dist.rank == 0 and not args.skip_schemes and args.config != "C5":
        line["schemes"] = compare_schemes(spec, policy, 3, device)
    if dist.rank == 0 and not args.skip_cpu_baseline:
        from oracle import oracle as O
        threads = O.default_threads()
        cspec, shrink = cpu_sample_spec(spec)
        times, ctotal = cpu_window(cspec, policy, 1, 2, 1, threads)
        per = statistics.fmean(times)
        line["cpu_baseline"] = {"value": round(ctotal / per / 1e9, 4), "unit": "GB/s", "cores": threads,
                                "kind": "port",
                                "sample": f"2 full {args.config} windows (copy-in, attach, resolve, scale, "
                                          "detach, copy-out) by oracle/cf_oracle.c on the host"
                                          + (f", leaves shortened {shrink}x to fit host RAM" if shrink > 1 else "")}
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    if flush is not None:
        flush.close()
    if twin is not None:
        twin.close()
    w.close()


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C2")
    ap.add_argument("--chunk-mb", type=int, default=32)
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--skip-chase", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="enqueue every window directly (no CUDA graph)")
    ap.add_argument("--skip-schemes", action="store_true", help="skip the 4-scheme drop-in API comparison")
    ap.add_argument("--single-buffer", action="store_true", help="e2e with one image (no step overlap)")
    ap.add_argument("--leaf-elems", type=int, default=0, help="override the leaf length (plumbing tests only)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    dist = Dist()
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
