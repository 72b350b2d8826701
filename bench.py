#!/usr/bin/env python
"""Benchmark: deep-copy + leaf-kernel effective GB/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the hot path over one synthetic object graph:
  * value  -- the graph already resident in HBM: relocation (attach) -> pointerchain resolve ->
              leaf kernel -> detach, graph bytes / device time (CUDA events, max over ranks);
  * e2e    -- the same through the C-ABI window from pinned HOST buffers: chunked H2D of the
              arena + relocation tables, the device work, and the D2H copy-back of the whole
              arena inside the timed region (the harness.py:369-373 metered window).
Default workload C2: DenseSpec(q=4, depth=3, n=4Mi) float32 leaves-only -- a depth-4 pointer
chain (3 Lnext hops + A) to each of 64 leaf arrays of 4Mi floats, 1 GiB of payload.  At N=1 the
line also carries the reference's own dtype (C2 in f64) and C1 / C3 / C4 summaries.
``--gpus N`` without torchrun re-launches itself under torch.distributed.run (one rank per GPU;
ranks beyond the visible GPUs share them).  Each rank processes its own config-shaped subtree
(weak scaling; C5: one 64 GiB tree cut by subtree, strong scaling); no data-path collective.
``--impl reference`` times the CPU restatement of the reference path (oracle/, all host cores) on
the same workload, rank 0 only: its ``value`` is the same resident step (attach -> resolve ->
scale -> detach on a buffer already holding the arena), its ``e2e`` the full window with the
copies.  That arm imports nothing from the product package.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "deep-copy+kernel effective GB/s (H2D and HBM % of roofline) at 1/2/4/8 B200"

# The workloads, as plain data shared by both arms.  graph_bytes / leaf_bytes:
# one tree (per GPU for weak scaling; the whole tree for C5) in the aligned-16 f32 arena, as the
# native planner lays it out (tests/test_bench.py pins these against the planner).
CONFIGS = {
    "C1": dict(kind="linear", args=(1, 1_000_000, "allinit_allused"), elem=4, leaf_only=False, policy="all_arrays",
               graph_bytes=4_000_032, leaf_bytes=4_000_000,
               desc="C1: depth-1 struct with one float32 leaf array of 1M elements"),
    "C2": dict(kind="dense", args=(4, 4 << 20, 3), elem=4, leaf_only=True, policy="all_leaves",
               graph_bytes=1_073_743_104, leaf_bytes=1_073_741_824,
               desc="C2: depth-4 pointer chain, dense q=4 layout, 64 leaf arrays x 4Mi float32 (leaves only)"),
    "C3": dict(kind="forest", args=(4, 4 << 20, "LLinit_LLused"), elem=4, leaf_only=False, policy="all_leaves",
               graph_bytes=1_073_750_008, leaf_bytes=1_073_741_824,
               desc="C3: 64 x depth-4 linear chains (LLinit_LLused), 64 leaves x 4Mi float32, 320 objects "
                    "scattered over the slab (seeded permutation)"),
    "C4": dict(kind="dense", args=(100, 256, 3), elem=4, leaf_only=False, policy="all_leaves",
               graph_bytes=1_046_585_856, leaf_bytes=1_024_000_000,
               desc="C4: 1,010,101 structs, 1M leaves x 256 float32, depth 3, relocation-bound"),
    "C5": dict(kind="dense", args=(4, 268_435_456, 3), elem=4, leaf_only=True, policy="all_leaves",
               graph_bytes=68_719_478_016, leaf_bytes=68_719_476_736,
               desc="C5: 64 GiB depth-4 dense graph (64 leaves x 256Mi float32), cut by subtree over the GPUs"),
}
FOREST = 64            # C3: chains per forest
C3_SCATTER = 0xC3
# working sets below this are L2-flushed before every timed step (B200 L2 = 126 MB)
L2_FLUSH_BELOW = 512 << 20
NOMINAL_HBM_GBS = 8000.0   # vendor figure, reported beside the measured-copy roofline
LINK_PROBE_BYTES = 1 << 30
# small graphs: e2e steps rotate over at least this many bytes of images (> the 126 MB L2; a ring
# of 34 C1 windows measured 0.85 of the same-size link, 68 windows 0.79: tools/c1_ring_probe.py)
RING_BYTES = 128 << 20


def scaling_of(name: str) -> str:
    return "strong" if name == "C5" else "weak"


def workload_config(name: str, world: int, leaf_elems: int = 0, elem: int = 4) -> dict:
    """The workload as both arms name it: identical keys and values (pure data)."""
    c = CONFIGS[name]
    graph, leaf = c["graph_bytes"], c["leaf_bytes"]
    n_full = c["args"][1]
    desc = c["desc"]
    if leaf_elems and leaf_elems < n_full:
        f = leaf_elems / n_full
        leaf = int(leaf * f)
        graph = graph - c["leaf_bytes"] + leaf   # nodes unchanged, leaves shortened (approximate padding)
        desc += f" [leaves shortened to {leaf_elems} elements: plumbing run, not a bench value]"
    if elem != c["elem"]:
        graph, leaf = graph + leaf * (elem // c["elem"] - 1), leaf * elem // c["elem"]
    scaling = scaling_of(name)
    per_gpu = graph if scaling == "weak" else graph // world
    return {"workload": desc, "graph_bytes_per_gpu": per_gpu,
            "leaf_bytes_per_gpu": leaf if scaling == "weak" else leaf // world,
            "dtype": "f32" if elem == 4 else "f64", "layout": "aligned16 arena (reference node layout)",
            "targets": c["policy"],
            "l2": ("inputs >= 1 GiB per GPU exceed the 126 MB L2 (no flush needed)" if per_gpu >= L2_FLUSH_BELOW else
                   "working set below 512 MiB: the GPU arm's e2e steps rotate over device images and copy-back "
                   f"buffers totalling >= {RING_BYTES >> 20} MiB (inputs larger than the 126 MB L2); its resident "
                   "steps are each preceded by an L2 flush (a read pass over a 512 MiB device buffer: clean lines, nothing "
                   "written back inside a step) outside the timed intervals"),
            "parallelism": f"dp{world} ({scaling}-scaled subtree shards, one per GPU, no data-path collective)"}


def make_spec(name: str, elem: int | None = None, leaf_elems: int = 0):
    """The config as a product-package spec (our arm only)."""
    from paper_1906_01128_b200 import DenseSpec, ForestSpec, LinearSpec
    c = CONFIGS[name]
    e = elem or c["elem"]
    args = list(c["args"])
    if leaf_elems and leaf_elems < args[1]:
        args[1] = leaf_elems
    if c["kind"] == "forest":
        spec = ForestSpec(LinearSpec(*args, elem=e), FOREST, scatter_seed=C3_SCATTER)
    elif c["kind"] == "linear":
        spec = LinearSpec(*args, elem=e)
    else:
        spec = DenseSpec(*args, elem=e, leaf_only=c["leaf_only"])
    return spec, c["policy"], c["desc"]


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

    def _reduce(self, x: float, op) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        return self._reduce(x, self.pg.ReduceOp.MAX) if self.pg else x

    def min(self, x: float) -> float:
        return self._reduce(x, self.pg.ReduceOp.MIN) if self.pg else x

    def sum(self, x: float) -> float:
        return self._reduce(x, self.pg.ReduceOp.SUM) if self.pg else x

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def share_host_threads(dist: "Dist") -> None:
    """torchrun pins OMP_NUM_THREADS=1 per rank; the native planner / builder (OpenMP, outside the
    timed regions) then fills a rank's arena on one core.  Give each rank its share of this
    process's CPUs instead (the oracle legs set their own thread counts)."""
    if dist.world <= 1:
        return
    import ctypes
    try:
        cpus = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        cpus = os.cpu_count() or 1
    local = int(os.environ.get("LOCAL_WORLD_SIZE", dist.world))
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(max(1, cpus // max(1, local)))
    except OSError:
        pass


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def respawn(args, argv) -> int:
    """``--gpus N`` (N > 1) outside torchrun: re-launch this script as N ranks, one per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()), *argv]
    return subprocess.run(cmd).returncode


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


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------------------ CPU legs
CPU_SAMPLE_BYTES = 2 << 30  # bound on the CPU legs' working set (3 buffers of this size)


def oracle_spec(name: str, elem: int, leaf_elems: int = 0):
    """(OSpec of one tree, trees per workload unit, leaf shortening factor) for the oracle port.
    Leaves are shortened so one CPU graph stays <= CPU_SAMPLE_BYTES; C3 is 64 chains."""
    from oracle import oracle as O
    c = CONFIGS[name]
    args = list(c["args"])
    if leaf_elems and leaf_elems < args[1]:
        args[1] = leaf_elems
    if c["kind"] == "dense":
        mk = lambda n: O.OSpec(O.DENSE, args[0], n, args[2], "allinit_allused", elem, c["leaf_only"], 16)  # noqa: E731
    else:
        mk = lambda n: O.OSpec(O.LINEAR, args[0], n, 0, args[2], elem, False, 16)  # noqa: E731
    spec = mk(args[1])
    trees = FOREST if c["kind"] == "forest" else 1
    total = int(O.counts(spec).total)
    if total <= CPU_SAMPLE_BYTES:
        return spec, trees, 1
    f = -(-total // CPU_SAMPLE_BYTES)
    return mk(args[1] // f), trees, f


class OracleLeg:
    """The oracle port of the reference window on the host cores (test infrastructure as the
    timed CPU baseline only): ``window`` = copy in, attach, resolve, scale, detach, copy out;
    ``resident`` = the same without the two copies."""

    def __init__(self, name: str, elem: int = 4, leaf_elems: int = 0, threads: int | None = None):
        from oracle import oracle as O
        self.O = O
        self.spec, self.trees, self.shrink = oracle_spec(name, elem, leaf_elems)
        self.threads = threads or O.default_threads()
        self.t = O.build(self.spec, 1)
        pol = {"ref": O.TARGET_REF, "all_leaves": O.TARGET_ALL_LEAVES,
               "all_arrays": O.TARGET_ALL_ARRAYS}[CONFIGS[name]["policy"]]
        self.idx = O.targets(self.t, pol)
        self.keys = O.chain_keys(self.t, self.idx)
        # one (arena, device buffer, copy-back buffer) per tree of the workload unit (C3: 64
        # chains), each its own memory -- re-running one small tree would time CPU-cache hits
        import dataclasses
        self.units = []
        for k in range(self.trees):
            t = self.t if k == 0 else dataclasses.replace(self.t, buf=self.t.buf.copy())
            self.units.append((t, t.buf.copy(), np.empty_like(t.buf)))
        self.dev_base = 0x7E00_0000_0000
        self.graph = self.t.total * self.trees

    def run(self, kind: str, steps: int, warmup: int, budget_s: float = 60.0) -> list:
        times = []
        for i in range(warmup + steps):
            s = 2.0 if i % 2 == 0 else 0.5
            t0 = time.perf_counter()
            for t, dev, out in self.units:
                if kind == "window":
                    rc = self.O.window(t, self.idx, dev, out, t.ptr_base, self.dev_base, s, self.threads, keys=self.keys)
                else:
                    rc = self.O.resident(t, self.idx, dev, t.ptr_base, self.dev_base, s, self.threads, keys=self.keys)
                if rc != -1:
                    raise RuntimeError(f"oracle {kind} reported site {rc}")
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
            if sum(times) > budget_s and len(times) >= 2:
                break
        return times

    def sample_text(self, name: str, what: str) -> str:
        return (f"{what} of {name} by oracle/cf_oracle.c (OpenMP, {self.threads} threads)"
                + (f", {self.trees} chains, each in its own memory" if self.trees > 1 else "")
                + (f", leaves shortened {self.shrink}x to bound host RAM (GB/s of the sample's graph bytes)"
                   if self.shrink > 1 else ""))


def reference_python_baseline(budget_s: float = 20.0) -> dict:
    """The unmodified reference (pip-installed into baseline/_ref, else /root/reference when present)
    timed on ONE core: its execute_case window transfer_to_device -> kernel_scale -> copy_back
    (harness.py:369-373), marshalling scheme, its own f64 and target policy.  C1 at full size;
    C2 (reference form: DenseSpec(4, n, 3), arrays on every node) with n reduced 64x, reported as
    GB/s of graph bytes (linear in n, labelled as an extrapolation)."""
    roots = [REPO / "baseline" / "_ref", Path("/root/reference/pkg/src")]
    root = next((r for r in roots if (r / "chainforge" / "__init__.py").exists()), None)
    if root is None:
        return {"kind": "reference_python", "unavailable": "reference package not installed (baseline/_ref)"}
    code = r'''
import json, sys, time
sys.path.insert(0, sys.argv[1])
import chainforge as cfr
from chainforge.harness import transfer_to_device, kernel_scale, copy_back
from chainforge.memory import Machine
from chainforge.scenarios import LinearSpec, DenseSpec, marshal_tree, tree_total_bytes
budget = float(sys.argv[2])
out = {}
for name, spec, note in (("C1", LinearSpec(1, 1_000_000, "allinit_allused"), "full size"),
                         ("C2", DenseSpec(4, (4 << 20) // 64, 3), "n reduced 64x (4Mi -> 64Ki), arrays on every node")):
    times = []
    t_all = time.perf_counter()
    while len(times) < 3 and (time.perf_counter() - t_all) < budget:
        m = Machine()
        arena, h = marshal_tree(m, spec, seed=1)
        t0 = time.perf_counter()
        prep = transfer_to_device(m, h, "marshalling", arena)
        kernel_scale(m, h, prep, 2.0)
        copy_back(m, h, prep)
        times.append(time.perf_counter() - t0)
    best = min(times)
    g = tree_total_bytes(spec)
    out[name] = {"window_s": round(best, 5), "graph_bytes": g, "gbs": round(g / best / 1e9, 5), "windows": len(times),
                 "sample": note}
print(json.dumps(out))
'''
    try:
        env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
        r = subprocess.run(["taskset", "-c", "0", sys.executable, "-c", code, str(root), str(budget_s)],
                           capture_output=True, text=True, timeout=10 * budget_s + 60, env=env)
        if r.returncode != 0:
            return {"kind": "reference_python", "unavailable": (r.stderr or r.stdout)[-200:]}
        res = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as exc:
        return {"kind": "reference_python", "unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    return {"kind": "reference_python", "value": res["C2"]["gbs"], "unit": "GB/s", "cores": 1,
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "sample": "unmodified reference execute_case window (marshalling, f64, its own target policy) on "
                      "1 core (taskset -c 0); value = C2 with n reduced 64x (GB/s of graph bytes, extrapolated "
                      "linearly to full n)", "configs": res, "source": str(root.relative_to(REPO))
            if root.is_relative_to(REPO) else str(root)}


def run_reference(args, dist: Dist) -> None:
    """The reference arm: the oracle port of the reference path on all host cores (rank 0 only)."""
    if dist.rank != 0:
        return
    leg = OracleLeg(args.config, CONFIGS[args.config]["elem"], args.leaf_elems)
    res = leg.run("resident", args.steps, args.warmup)
    win = leg.run("window", args.steps, args.warmup)
    r_per, w_per = statistics.fmean(res), statistics.fmean(win)
    value = leg.graph / r_per / 1e9
    e2e = leg.graph / w_per / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": len(res), "warmup": args.warmup,
        "ms_per_step": round(r_per * 1e3, 3), "higher_is_better": True, "scaling": scaling_of(args.config),
        "vs_baseline": None, "dtype": "f32" if leg.spec.elem == 4 else "f64",
        "data": "synthetic (payload_values of the reference, seed 1)",
        "config": workload_config(args.config, args.gpus, args.leaf_elems),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": leg.threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": leg.sample_text(args.config, "resident step (attach, resolve, scale, detach on a "
                                                                 "buffer already holding the arena)")},
        "e2e": {"value": round(e2e, 4), "unit": "GB/s", "ms_per_step": round(w_per * 1e3, 3),
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "what": leg.sample_text(args.config, "full window (copy in, attach, resolve, scale, detach, copy out)")},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def verify_gather(w, shard, spec, dist: Dist, device: int, ndev: int, src_factor: float) -> dict:
    """Outside the timed region: one more window (scale 2.0) from the host arena, per-leaf
    position-weighted checksums of the device image (cf_checksum_ranges), all-gathered to every
    rank -- over NCCL when each rank has its own GPU, else gloo -- and checked on rank 0 against
    the checksums of the whole workload (payload_values * factor, the same for every leaf of a
    level)."""
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
    # one tree cut by subtree: keys are the whole tree's leaf ordinals, one seed; otherwise every
    # rank owns a tree of its own (seed + rank): keys are (rank, position)
    per_rank_trees = not shard.whole_tree
    keys = (np.arange(len(tg), dtype=np.int64) + np.int64(dist.rank) * (1 << 32)) if per_rank_trees \
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
    out = {"backend": backend, "leaves": int(len(o)), "what": "per-leaf position-weighted u32-word checksums after "
           "a verification window (scale 2.0), gathered to all ranks"}
    if err:
        out["nccl_error"] = err
    if dist.rank == 0:
        f = 2.0 * src_factor
        ok = True
        memo = {}
        lv, n = int(lvl[tg[0]]), int(cnt[tg[0]])
        for key, val in zip(o.tolist(), v.tolist()):
            seed = shard.base_seed + (key >> 32) if per_rank_trees else shard.seed
            if seed not in memo:
                memo[seed] = expected_checksum(seed, lv, n, spec.elem, f)
            ok &= int(val) == memo[seed]
        want = dist.world * len(tg) if per_rank_trees else int(spec.q ** spec.depth)
        out["complete"] = int(len(o)) == want and len(set(o.tolist())) == len(o)
        out["checksums_match"] = bool(ok)
        if not (ok and out["complete"]):
            raise SystemExit(f"gathered result check failed: {out}")
    return out


class L2Flush:
    """Evicts the L2 between timed steps (a read pass over a 512 MiB device buffer on the window's
    stream, outside the timed intervals: the L2 is left holding clean lines, so nothing of the
    flush is written back inside a timed step) and times each step on the device (CUDA events
    inside the window)."""

    def __init__(self, w):
        import ctypes as C

        from paper_1906_01128_b200 import _native as N
        self.N, self.w = N, w
        self.buf = C.c_void_p()
        N.check(N.lib().cf_dev_alloc(w.ctx.handle, L2_FLUSH_BELOW, C.byref(self.buf)))
        N.check(N.lib().cf_memset(w.ctx.handle, self.buf, 0x5A, L2_FLUSH_BELOW))   # defined contents

    def flush(self) -> None:
        self.N.check(self.N.lib().cf_l2_evict(self.w.ctx.handle, self.buf, L2_FLUSH_BELOW))

    def steps(self, flags: int, n: int):
        return self.w.run_n_flushed(n, self.buf.value, L2_FLUSH_BELOW, flags=flags)

    def close(self) -> None:
        self.N.lib().cf_dev_free(self.w.ctx.handle, self.buf)


class Measured:
    """One workload measured on this rank's GPU: links, e2e, resident step, leaf kernel, chase."""

    def __init__(self, spec, policy: str, seed: int, device: int, chunk_mb: int, numa_node: int,
                 single_buffer: bool = False, graph: bool = True):
        from paper_1906_01128_b200 import DeepCopyWindow
        from paper_1906_01128_b200 import _native as N
        self.N = N
        t0 = time.perf_counter()
        self.w = w = DeepCopyWindow(spec, seed=seed, policy=policy, mode="resolved", align=16, numa_node=numa_node,
                                    chunk_bytes=chunk_mb << 20, device=device,
                                    separate_output=spec.n * spec.elem * 64 <= (16 << 30))
        self.build_s = time.perf_counter() - t0
        self.spec = spec
        self.total = w.total
        # small graphs (C1: 4 MB): two steps of at least 1 MiB, so copy-out of the first half
        # overlaps copy-in of the second (measured: 0.173 -> 0.156 ms per C1 window)
        if self.total <= 4 * w.chunk_bytes:
            w.chunk_bytes = min(w.chunk_bytes, max(1 << 20, ((self.total + 1) // 2 + (1 << 20) - 1) >> 20 << 20))
        self.leaf_bytes = int(sum(int(w.plan.table(N.CF_TAB_ARR_COUNT)[i]) for i in w.targets)) * spec.elem
        self.kernel_traffic = 2 * self.leaf_bytes   # read + write of every targeted element
        # double-buffered: two windows over the same arena, own images / copy-back buffers, so step
        # r+1 copies in while step r copies out (skipped when two images would not fit)
        self.twin = w.twin() if (w.dst != w.src and not single_buffer) else None
        self.gflag = N.CF_WIN_GRAPH if graph else 0
        self.flush = L2Flush(w) if self.total < L2_FLUSH_BELOW else None
        # small graphs: windows with copies rotate over a ring of images / copy-back buffers larger
        # than the L2, so consecutive steps overlap without finding earlier steps' data cached
        self.ring = []
        if self.flush is not None and self.twin is not None:
            k = max(2, -(-RING_BYTES // self.total))
            self.ring = [self.twin] + [w.twin() for _ in range(k - 2)]

    def _run_n(self, flags: int, n: int):
        w = self.w
        if flags & (self.N.CF_WIN_H2D | self.N.CF_WIN_D2H):
            if self.ring:
                return w.run_ring_n(self.ring, n, flags=flags)
            if self.twin is not None:
                return w.run_pair_n(self.twin, n, flags=flags)
        return w.run_n(n, flags=flags)

    def pipeline_link(self, dist: Dist) -> dict:
        """Copy-only windows with the e2e window's own chunking and buffering (second denominator)."""
        N, link = self.N, {}
        for name, fl in (("h2d", N.CF_WIN_H2D), ("d2h", N.CF_WIN_D2H), ("bidir", N.CF_WIN_H2D | N.CF_WIN_D2H)):
            self._run_n(fl, 2)
            dist.barrier()
            st = self._run_n(fl, 4)
            link[name] = (st.h2d_bytes + st.d2h_bytes) / (st.ms_total * 1e-3) / 1e9
        return link

    def timed(self, flags: int, warmup: int, steps: int, dist: Dist):
        """W warm-up windows, then K timed ones between barriers: (stats, host wall seconds from the
        common start barrier to this rank's completion)."""
        N = self.N
        copies = flags & (N.CF_WIN_H2D | N.CF_WIN_D2H)
        if self.flush is not None and not (copies and self.ring):
            self.flush.steps(flags, warmup)
            dist.barrier()
            t0 = time.perf_counter()
            st = self.flush.steps(flags, steps)
            wall = time.perf_counter() - t0
            dist.barrier()
            return st, wall
        if copies and self.ring:   # prime: every ring window captures its CUDA graph before the warm-up
            self._run_n(flags, len(self.ring) + 1)
        self._run_n(flags, warmup)
        N.check(N.lib().cf_ctx_sync(self.w.ctx.handle))
        dist.barrier()
        t0 = time.perf_counter()
        st = self._run_n(flags, steps)
        N.check(N.lib().cf_ctx_sync(self.w.ctx.handle))
        wall = time.perf_counter() - t0
        dist.barrier()
        return st, wall

    def kernel_ms(self, n: int, mode: str = "resolved") -> tuple[float, float]:
        """Leaf-kernel duration (events around the k_scale launch on the window's stream), resident,
        after one warm-up: (mean kernel ms, mean resident-step ms)."""
        self.w.run_resident(scale=2.0, mode=mode)
        ks, ts = [], []
        for i in range(n):
            if self.flush is not None:
                self.flush.flush()
            s = self.w.run_resident(scale=2.0 if i % 2 == 0 else 0.5, mode=mode)
            ks.append(s.ms_kernel)
            ts.append(s.ms_total)
        return statistics.fmean(ks), statistics.fmean(ts)

    @property
    def e2e_layout(self) -> str:
        if self.ring:
            return f"ring of {len(self.ring) + 1} windows ({(len(self.ring) + 1) * self.total >> 20} MiB of images)"
        return "double-buffered pair" if self.twin is not None else "single window"

    def close(self):
        if self.flush is not None:
            self.flush.close()
        for t in self.ring[1:]:
            t.close()
        if self.twin is not None:
            self.twin.close()
        self.w.close()


def plain_link(ctx, nbytes: int, iters: int = 1) -> dict:
    """Plain cudaMemcpyAsync probe, best of several repetitions (small sizes vary run to run:
    more repetitions for them)."""
    from paper_1906_01128_b200 import _native as N
    reps = 3 if nbytes >= (256 << 20) else 10
    return {k: round(v, 2) for k, v in N.link_probe(ctx, nbytes, iters=iters, reps=reps).items()}


def summary_block(name: str, elem: int, device: int, chunk_mb: int, numa_node: int, steps: int, warmup: int,
                  dist: Dist, peaks: dict, link_1g: dict) -> dict:
    """A compact line for one more workload on this GPU (N=1): resident step, leaf-kernel roofline
    fraction, e2e GB/s and its fraction of the independent link probe."""
    spec, policy, _ = make_spec(name, elem=elem)
    m = Measured(spec, policy, 1, device, chunk_mb, numa_node)
    N = m.N
    if m.total < (64 << 20):
        # small graphs (C1: 0.1 ms windows): >= 100 windows, so the batch's pipeline fill and drain
        # (one window's copy-in before any copy-out, and the reverse at the end) stay a small share
        steps = max(steps, 100)
    try:
        # small graphs: three batches, the median one reported (a 0.1 ms window is sensitive to
        # host-side hiccups of a single batch; all three are in the block)
        batches = 3 if m.total < (64 << 20) else 1
        runs = []
        for _ in range(batches):
            st, _w = m.timed(N.CF_WIN_FULL | m.gflag, warmup, steps, dist)
            runs.append((st.ms_total / steps, st))
        e2e_ms, st_e2e = sorted(runs, key=lambda r: r[0])[len(runs) // 2]
        m.w.upload_raw()
        st_res, _ = m.timed(N.CF_WIN_RESIDENT | m.gflag, warmup, steps, dist)
        res_ms = st_res.ms_total / steps
        k_ms, _ = m.kernel_ms(max(5, steps // 2))
        table = table_resolve_block(m, name, warmup, steps, dist, res_ms)
        h2d, d2h = st_e2e.h2d_bytes // steps, st_e2e.d2h_bytes // steps
        probe = link_1g if m.total >= (64 << 20) else plain_link(m.w.ctx, m.total, iters=8)
        ideal = (h2d + d2h) / (probe["bidir"] * 1e9) * 1e3
        achieved = m.kernel_traffic / (k_ms * 1e-3) / 1e9
        return {"workload": CONFIGS[name]["desc"] + ("" if elem == CONFIGS[name]["elem"] else " [float64]"),
                "dtype": "f32" if elem == 4 else "f64", "graph_bytes": m.total,
                "resident_ms_per_step": round(res_ms, 4), "value_gbs": round(m.total / (res_ms * 1e-3) / 1e9, 2),
                "kernel_ms": round(k_ms, 4), "kernel_hbm_gbs": round(achieved, 1),
                "kernel_frac": round(achieved / peaks["hbm_gbs"], 4),
                "kernel_share_of_resident_step": round(k_ms / res_ms, 4),
                "e2e_ms_per_step": round(e2e_ms, 4), "e2e_gbs": round(m.total / (e2e_ms * 1e-3) / 1e9, 3),
                "steps": steps,
                **({"e2e_batches_ms_per_step": [round(r[0], 4) for r in runs], "e2e_batch": "median of 3"}
                   if batches > 1 else {}),
                "link_probe_gbs": probe, "link_probe_bytes": LINK_PROBE_BYTES if probe is link_1g else m.total,
                "frac_of_link_roofline": round(ideal / e2e_ms, 4),
                "e2e_windows": m.e2e_layout,
                **({"table_resolve": table} if table else {})}
    finally:
        m.close()


def table_resolve_block(m, name: str, warmup: int, steps: int, dist, res_ms: float) -> dict:
    """C4 (many small leaves): the same resident step planned without leaf ownership
    (CF_WIN_TABLE_RESOLVE: every leaf resolved into the EA table, every site listed) -- the
    table-driven design the leaf-owned step replaces, timed in the same run."""
    if name != "C4":
        return {}
    N = m.N
    m.w.upload_raw()
    st, _ = m.timed(N.CF_WIN_RESIDENT | N.CF_WIN_TABLE_RESOLVE | m.gflag, warmup, steps, dist)
    t_ms = dist.max(st.ms_total) / steps
    m.w.upload_raw()
    return {"resident_ms_per_step": round(t_ms, 4), "leaf_owned_resident_ms_per_step": round(res_ms, 4),
            "what": "resident step planned with CF_WIN_TABLE_RESOLVE (EA table + full site list) vs the "
                    "leaf-owned step of this line"}


def run_ours(args, dist: Dist) -> None:
    from paper_1906_01128_b200 import _native as N
    from paper_1906_01128_b200.shard import shard_for

    ndev = N.device_count()
    if ndev == 0:
        raise SystemExit("no CUDA device visible: the product path has no CPU fallback")
    # one rank per GPU; ranks beyond the visible GPUs share them (plumbing runs on small boxes)
    device = dist.local_rank % ndev
    spec, policy, _ = make_spec(args.config, leaf_elems=args.leaf_elems)
    scaling = scaling_of(args.config)
    shard = shard_for(spec, dist.rank, dist.world, scaling)
    spec = shard.spec
    # pinned arenas next to this GPU's host link (multi-socket boxes)
    numa_node = N.gpu_numa_node(device)
    m = Measured(spec, policy, shard.seed, device, args.chunk_mb, numa_node, args.single_buffer, not args.no_graph)
    w = m.w
    peaks = measured_peaks()

    # host-link denominators, every rank probing at once (the concurrent per-GPU link peak):
    # (1) plain cudaMemcpyAsync of 1 GiB, (2) copy-only windows shaped like the e2e pipeline,
    # (3) for small graphs, plain copies of the graph's own size back to back
    dist.barrier()
    link_plain = plain_link(w.ctx, LINK_PROBE_BYTES)
    dist.barrier()
    link_pipe = m.pipeline_link(dist)
    link_small = None
    if m.total < (64 << 20):
        dist.barrier()
        link_small = plain_link(w.ctx, m.total, iters=8)

    clocks = ClockSampler(device)
    clocks.start()
    # ---- e2e: host buffers in, copy-back out, through the C-ABI window
    st_e2e, wall_e2e = m.timed(N.CF_WIN_FULL | m.gflag, args.warmup, args.steps, dist)
    e2e_ms = dist.max(st_e2e.ms_total) / args.steps
    e2e_wall_ms = dist.max(wall_e2e) * 1e3 / args.steps
    # ---- value: image resident in HBM
    w.upload_raw()
    st_res, wall_res = m.timed(N.CF_WIN_RESIDENT | m.gflag, args.warmup, args.steps, dist)
    res_ms = dist.max(st_res.ms_total) / args.steps
    res_wall_ms = dist.max(wall_res) * 1e3 / args.steps
    # ---- leaf-kernel duration (events around the k_scale launch, resident, after warm-up)
    kernel_ms, _ = m.kernel_ms(max(5, args.steps // 2))
    # ---- C4: the table-driven resident step (no leaf ownership) beside it
    table = table_resolve_block(m, args.config, args.warmup, args.steps, dist, res_ms) if not args.leaf_elems else {}
    # ---- chase-per-access comparison (same resident image)
    chase = {}
    if not args.skip_chase:
        c_ms, c_step = m.kernel_ms(4, mode="chase")
        chase = {"kernel_ms": round(c_ms, 4), "hbm_gbs": round(m.kernel_traffic / (c_ms * 1e-3) / 1e9, 1),
                 "resident_ms_per_step": round(c_step, 4)}
    clk = clocks.stop()

    # correctness spot check of the copy-back on the first and last targeted leaf
    arr, cnt, lvl = w.plan.table(N.CF_TAB_ARR_OFF), w.plan.table(N.CF_TAB_ARR_COUNT), w.plan.table(N.CF_TAB_ARR_LEVEL)
    dt = np.float32 if spec.elem == 4 else np.float64
    ring = [w] + (m.ring or ([m.twin] if m.twin is not None else []))
    last = ring[(args.steps - 1) % len(ring)]
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
    graph_all = dist.sum(float(m.total))
    value = graph_all / (res_ms * 1e-3) / 1e9
    e2e = graph_all / (e2e_ms * 1e-3) / 1e9
    achieved = m.kernel_traffic / (kernel_ms * 1e-3) / 1e9
    h2d_step = st_e2e.h2d_bytes // args.steps
    d2h_step = st_e2e.d2h_bytes // args.steps
    denom = link_small or link_plain
    ideal_ms = (h2d_step + d2h_step) / (denom["bidir"] * 1e9) * 1e3
    ideal_pipe_ms = (h2d_step + d2h_step) / (link_pipe["bidir"] * 1e9) * 1e3
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(res_ms, 4), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32" if spec.elem == 4 else "f64",
        "data": "synthetic (payload_values of the reference, seed 1+rank)",
        "config": workload_config(args.config, n, args.leaf_elems),
        "pipeline": {"chunk_bytes": w.chunk_bytes, "h2d_streams": 1, "d2h_streams": 1, "cuda_graph": not args.no_graph,
                     "e2e_windows": m.e2e_layout,
                     "l2_flushed_before_resident_steps": m.flush is not None,
                     "graph_bytes_this_rank": m.total, "leaf_bytes_this_rank": m.leaf_bytes},
        "value_host_wall": {"value": round(graph_all / (res_wall_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                            "ms_per_step": round(res_wall_ms, 4),
                            "what": "all ranks' graph bytes / host wall time from the common start barrier to the "
                                    "last rank's completion (max over ranks), per step"},
        "e2e": {"value": round(e2e, 3), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": int(h2d_step), "d2h_bytes_per_step": int(d2h_step),
                "host_wall_gbs": round(graph_all / (e2e_wall_ms * 1e-3) / 1e9, 3),
                "host_link_gbs": link_plain,
                "host_link_probe": f"plain cudaMemcpyAsync of {LINK_PROBE_BYTES >> 20} MiB pinned<->HBM (cf_link_probe), "
                                   "all ranks probing at once, best of 3",
                "host_link_same_size_gbs": link_small,
                "ideal_ms_at_measured_bidir": round(ideal_ms, 3),
                "frac_of_link_roofline": round(ideal_ms / e2e_ms, 4),
                "pipeline_link_gbs": {k: round(v, 2) for k, v in link_pipe.items()},
                "frac_of_pipeline_link": round(ideal_pipe_ms / e2e_ms, 4),
                "gpu_launches_per_step": int(st_e2e.launches // args.steps),
                "windows": m.e2e_layout},
        "roofline": {"bound": "hbm", "kernel": f"k_scale<{'float' if spec.elem == 4 else 'double'},resolved>",
                     "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "peak_source": peaks["source"],
                     "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                     "traffic": ncu_record(args.config).get("dram_bytes_per_launch"),
                     "frac_of_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                     "ncu_dram_pct_of_peak": ncu_record(args.config).get("dram_pct_of_ncu_peak"),
                     "algorithmic_bytes_per_launch": m.kernel_traffic, "kernel_ms": round(kernel_ms, 4),
                     "share_of_resident_step": round(kernel_ms / res_ms, 4)},
        "modes": {"resolved": {"kernel_ms": round(kernel_ms, 4), "hbm_gbs": round(achieved, 1)}, "chase": chase,
                  **({"table_resolve": table} if table else {})},
        "gpu_launches": int(st_res.launches),
        "numa": {"gpu_node": numa_node, "host_arenas": "allocated on the GPU's node" if numa_node >= 0 else "OS placement"},
        "gather": gather,
        "clocks": clk,
        "build_s": round(m.build_s, 2),
    }
    m.close()
    extras = n == 1 and not args.skip_extras and not args.leaf_elems
    if extras and args.config == "C2":
        # the reference's own dtype (float64, scenarios.py:22): C2 with 2 GiB of f64 leaves
        line["f64"] = summary_block("C2", 8, device, args.chunk_mb, numa_node, min(args.steps, 10), args.warmup,
                                    dist, peaks, link_plain)
    if extras:
        line["per_config"] = {}
        for name in ("C1", "C2", "C3", "C4"):
            if name != args.config:
                line["per_config"][name] = summary_block(name, 4, device, args.chunk_mb, numa_node,
                                                         min(args.steps, 10), args.warmup, dist, peaks, link_plain)
        # the reference's own dtype on the relocation-bound shape too (1M leaves of 256 float64)
        line["per_config"]["C4_f64"] = summary_block("C4", 8, device, args.chunk_mb, numa_node, min(args.steps, 10),
                                                     args.warmup, dist, peaks, link_plain)
    if dist.rank == 0 and not args.skip_schemes and args.config != "C5":
        line["schemes"] = compare_schemes(spec, policy, 3, device)
    if dist.rank == 0 and not args.skip_cpu_baseline:
        leg = OracleLeg(args.config, spec.elem, args.leaf_elems)
        times = leg.run("window", 2, 1, budget_s=30.0)
        line["cpu_baseline"] = {"value": round(leg.graph / statistics.fmean(times) / 1e9, 4), "unit": "GB/s",
                                "cores": leg.threads, "kind": "port", "cpu_model": cpu_model(),
                                "sample": leg.sample_text(args.config, f"{len(times)} full windows (copy-in, attach, "
                                                          "resolve, scale, detach, copy-out)")}
        line["cpu_baseline_reference_python"] = reference_python_baseline()
    if dist.rank == 0:
        print(json.dumps(line), flush=True)


def compare_schemes(spec, policy: str, reps: int, device: int) -> dict:
    """The four transfer schemes of the reference (harness.py:219-325) through the drop-in API on
    the same graph: window = transfer_to_device -> kernel_scale -> copy_back, host wall clock
    with device syncs, median of `reps` after one warm-up.  UVM is measured without hints, with a
    pipelined chunked prefetch, and with each advice; GB/s are graph bytes over the window."""
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


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C2")
    ap.add_argument("--chunk-mb", type=int, default=32)
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--skip-chase", action="store_true")
    ap.add_argument("--skip-extras", action="store_true", help="skip the f64 and per-config summary blocks")
    ap.add_argument("--no-graph", action="store_true", help="enqueue every window directly (no CUDA graph)")
    ap.add_argument("--skip-schemes", action="store_true", help="skip the 4-scheme drop-in API comparison")
    ap.add_argument("--single-buffer", action="store_true", help="e2e with one image (no step overlap)")
    ap.add_argument("--leaf-elems", type=int, default=0, help="override the leaf length (plumbing tests only)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        raise SystemExit(respawn(args, argv))
    if world is not None and int(world) != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    dist = Dist()
    share_host_threads(dist)
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
