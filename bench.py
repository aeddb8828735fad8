"""Benchmark of the sparse-TTV hot path on B200 (one JSON line on rank 0).

Headline workload: BASELINE config 5 -- skewed 3-way COO tensor 1e6 x 1e5 x 1e4 with
4e8 distinct Zipf(1.2) coordinates, N(0,1) values, contracted in mode 2 (0-based) with a
uniform length-1e4 vector; sparse 1e6 x 1e5 result.  A "step" is one full TTV over the
tensor (all ranks' shards) through the C ABI (tk_ttv_f64_device), including the host
read-back of the result count.  Inputs (12.8 GB) exceed the 126 MB L2, so no flush is
needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--nnz NNZ] [--no-secondary] [--no-e2e] [--no-cpu]

--gpus N > 1: one process per GPU over NCCL.  Under torchrun (WORLD_SIZE set) WORLD_SIZE must
equal N; launched directly, bench.py starts torch.distributed.run itself with N ranks, and fails
if fewer than N GPUs are visible (TK_BENCH_ONE_GPU=1 + TK_BENCH_BACKEND=gloo: path check with
every rank on device 0, never a measurement).  nnz are sharded at key changes
(multi.shard_bounds); the merge is an all-gather of per-rank counts inside the timed region; time
= max over ranks of device time (CUDA events).

--impl reference: the reference's own compiled TTV (oracle/_ref, built from /root/reference's
.pyx) on every host thread over the SAME config-5 tensor, built on the host by the generator's
host twin (oracle/tk_gen_host.cpp, byte-identical to the device generator); the product package
is never imported on that path.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CFG5 = {"shape": (10**6, 10**5, 10**4), "nnz": 4 * 10**8, "k": 2, "zipf_s": 1.2, "seed": 12345, "xseed": 777}
CFG4 = {"shape": (20000,) * 4, "nnz": 10**8, "keep": 0, "seed": 4444}
METRIC = "sparse TTV throughput (config 5, skewed Zipf 4e8 nnz)"
WORKLOAD = "cfg5_ttv_zipf_1e6x1e5x1e4_nnz4e8_mode2"


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region.

    Reads the same NVML counters nvidia-smi prints (clocks.sm, clocks.max.sm,
    clocks_event_reasons.*) from a background thread every ~2 ms, so even a timed region
    of a few tens of milliseconds gets samples.
    """

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples = []
        self._stop = threading.Event()
        self._thr = None
        self._nv = None

    def _handle(self):
        """NVML handle of CUDA device `index`, matched by PCI bus id (NVML and CUDA orders can
        differ, e.g. under CUDA_VISIBLE_DEVICES), else by index."""
        nv = self._nv
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:  # noqa: BLE001
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _loop(self):
        nv = self._nv
        h = self._h
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, [n for n, bit in names.items() if r & bit]))
            except Exception:  # noqa: BLE001 - sampling must never break the bench
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = self._handle()  # resolved before the timed region starts
            self._thr = threading.Thread(target=self._loop, daemon=True)
            self._thr.start()
            time.sleep(0.01)
        except Exception:  # noqa: BLE001
            self._nv = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr is not None:
            self._thr.join(timeout=2)
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "nvml"}
        sm = [s[0] for s in self.samples]
        reasons = sorted({r for s in self.samples for r in s[2]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(s[1] for s in self.samples)),
                "reasons": reasons, "samples": len(sm), "source": "nvml (nvidia-smi counters), 2 ms period"}


# ---- process topology --------------------------------------------------------------------------

def launch_ranks(args) -> int:
    """``--gpus N`` without torchrun: start N ranks with torch.distributed.run (one process per
    GPU, NCCL).  Fails if fewer than N GPUs are visible, unless the one-GPU path check is asked
    for (TK_BENCH_ONE_GPU=1)."""
    import torch
    n = args.gpus
    have = torch.cuda.device_count()
    if have < n and os.environ.get("TK_BENCH_ONE_GPU") != "1":
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have} "
              "(TK_BENCH_ONE_GPU=1 TK_BENCH_BACKEND=gloo runs a path check on one GPU)", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # TK_BENCH_ONE_GPU=1 + TK_BENCH_BACKEND=gloo: path check only -- every rank on device 0,
        # collectives on the host (no kernel waits on another rank); never a measurement
        dev = 0 if os.environ.get("TK_BENCH_ONE_GPU") == "1" else local
        if dev >= torch.cuda.device_count():
            raise SystemExit(f"rank {rank}: device {dev} not visible ({torch.cuda.device_count()} GPUs)")
        torch.cuda.set_device(dev)
        backend = os.environ.get("TK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def make_comm(rank, world):
    """The data-plane communicator: NCCL inside libtk_b200.so (multi.NcclComm; torch.distributed
    only broadcasts its id).  The one-GPU path check (TK_BENCH_BACKEND=gloo) uses the gloo
    stand-in of the tests instead -- NCCL cannot put two ranks on one GPU."""
    if world == 1:
        return None
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        sys.path.insert(0, os.path.join(REPO, "tests"))
        from gloo_comm import GlooComm
        return GlooComm()
    from paper_2510_01495_b200 import multi
    return multi.NcclComm(rank, world)


def max_over_ranks(v: float, world: int) -> float:
    """Max of a host scalar over ranks (harness bookkeeping after the timed region)."""
    if world == 1:
        return v
    import torch.distributed as dist
    box = [None] * world
    dist.all_gather_object(box, float(v))
    return max(box)


def cpu_info():
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count()
    return os.cpu_count(), aff


def digest(subs, vals) -> dict:
    """sha256 of a TTV result's row-major subs and vals bytes (oracle.result_digest's definition)."""
    return {"u": int(len(vals)), "subs_sha256": hashlib.sha256(np.ascontiguousarray(subs).data).hexdigest(),
            "vals_sha256": hashlib.sha256(np.ascontiguousarray(vals).data).hexdigest()}


# ---- reference arm -----------------------------------------------------------------------------

def run_reference(args):
    """The reference's compiled ttv_raw (oracle/_ref) on the full config-5 tensor, on every host
    thread: the tensor is cut into one key-aligned shard per thread (oracle.shard_bounds; the
    concatenation is the one-call result) and each shard runs ``ttv_raw(..., release_gil=True)``
    on its own thread.  Operands come from the host twin of the device generator, so this is the
    same tensor our arm generates on the GPU (tests/test_gen_twin.py).  Only oracle/ is used."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle  # CPU reference arm: oracle/_ref + the host twin generator only
    cfg = CFG5
    nnz = args.nnz or cfg["nnz"]
    shape, k = cfg["shape"], cfg["k"]
    ncpu, threads = cpu_info()
    t0 = time.perf_counter()
    subs, vals = oracle.gen_coo(shape, nnz, zipf_s=cfg["zipf_s"], normal_vals=True, seed=cfg["seed"],
                                threads=threads)
    gen_s = time.perf_counter() - t0
    x = oracle.gen_uniform(shape[k], cfg["xseed"])
    times, parts, kind = [], None, "port"
    for i in range(args.warmup + args.steps):
        parts = None
        parts, el, kind = oracle.ttv_raw_threads(subs, vals, shape, x, k, threads)
        if i >= args.warmup:
            times.append(el)
    res = oracle.result_digest(parts)
    parts = None
    # one thread, one call (the reference's own self-timed ttv_timed) on a key-aligned prefix
    single = None
    ck = oracle.reference_module()
    if ck is not None:
        cut = oracle.shard_bounds(subs, 2, 8)[1]
        (_, _, _), el1 = ck.ttv_timed(subs[:cut], vals[:cut], shape, x, k)
        single = {"value": cut / el1, "unit": "nnz/s", "cores": 1, "seconds": el1,
                  "sample": f"first {cut} rows (1/8 of the tensor, cut at a key change), one ttv_timed call"}
    ms = 1e3 * float(np.mean(times))
    value = nnz / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (host twin of the device generator, seeded; byte-identical tensor)",
        "config": {"workload": WORKLOAD, "nnz": nnz, "shape": list(shape), "mode": k, "same_config": nnz == cfg["nnz"],
                   "gen_seconds": round(gen_s, 1), "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads, "kind": kind,
                         "sample": f"the full config-5 tensor ({nnz} rows) every step: {threads} key-aligned "
                                   f"shards on {threads} threads, ttv_raw(..., release_gil=True) each",
                         "host_cpus": ncpu, "affinity": threads, "single_core": single},
        "result": res,
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm: parity and CPU baselines (oracle = checker / baseline only) -----------------------

def host_tensor(t):
    """Row-major (nnz, d) int64 subs and float64 vals of a DeviceCoo, on the host (pageable)."""
    import torch
    subs = torch.stack(t.cols, dim=1).cpu().numpy()
    return np.ascontiguousarray(subs), t.vals.cpu().numpy()


def parity_cfg5(subs_h, vals_h, shape, xh, k, gpu_subs, gpu_vals, threads):
    """The full config-5 result of the GPU against the reference's own kernel (oracle/_ref) on
    the same tensor, bit for bit; the reference run is also the full-size CPU baseline."""
    from oracle import oracle
    parts, el, kind = oracle.ttv_raw_threads(subs_h, vals_h, shape, xh, k, threads)
    ok = oracle.compare_parts(parts, gpu_subs, gpu_vals)
    u_ref = sum(len(p[1]) for p in parts)
    return {"rows": int(subs_h.shape[0]), "u": u_ref, "bit_exact": bool(ok), "checked_against": kind,
            "seconds": el, "threads": threads}


def harness_baselines(threads):
    """Configs 1-3 through the reference's own harness (oracle/_ref: tenkern.run_experiment with
    its operand schedule, 30 measured trials + 1 warm-up): ``native-loop`` (the compiled kernels,
    one core), ``host-vectorized`` (tenhost's numpy TTV, config 3, 3 trials) and ``b200`` (this
    package registered in the same registry, so operands and clocks are the reference's)."""
    from oracle import oracle
    if oracle.reference_module() is None or not os.path.isdir(os.path.join(oracle.REF_DIR, "tenhost")):
        return None
    import tenkern
    from paper_2510_01495_b200 import registry
    registry.register()
    out = {}
    plan = [("cfg1_dot", tenkern.ExperimentConfig("dot", sizes=(10**6,), n_trials=30), ["native-loop", "b200"]),
            ("cfg2_matvec", tenkern.ExperimentConfig("matvec_square", sizes=(4096,), n_trials=30),
             ["native-loop", "b200"]),
            ("cfg3_ttv", tenkern.ExperimentConfig("ttv", sizes=(1000,), density=0.001, mode=3, n_trials=30),
             ["native-loop", "b200"]),
            ("cfg3_ttv_vectorized", tenkern.ExperimentConfig("ttv", sizes=(1000,), density=0.001, mode=3,
                                                             n_trials=3), ["host-vectorized"])]
    for name, cfg, labels in plan:
        recs = tenkern.run_experiment(cfg, labels)
        for s in tenkern.summarize(recs):
            out.setdefault(name, {})[s.implementation] = {"mean_s": s.mean_s, "sd_s": s.sd_s, "n": s.n,
                                                          "cores": 1 if s.implementation != "b200" else None}
    return out


def secondary_measurements(rank, steps, threads, with_cpu):
    """Configs 1-4 on one GPU (kernel time by CUDA events, L2 flushed between iterations by
    writing and then reading a 256 MB buffer), each with its parity against the reference's own
    kernels (oracle/_ref) on the same operands and, with ``with_cpu``, its CPU baseline."""
    import torch
    from oracle import oracle
    from paper_2510_01495_b200 import _lib, synth
    from paper_2510_01495_b200 import device as dv
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    lib = _lib.load()
    ck = oracle.reference_module()
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")  # 256 MB > 126 MB L2
    flush_sink = torch.empty((), dtype=torch.float64, device="cuda")
    res = {}

    def kernel_ms(fn):
        ts = []
        for i in range(steps + 2):
            torch.cuda.synchronize()
            flush.zero_()  # write 256 MB, then read it back: L2 is flushed and holds clean lines,
            flush_sink.copy_(flush.sum())  # so the timed kernel does not pay the write-back
            # no sync here: the call's start event and kernels queue behind the flush on the same
            # stream, so the host-side launch latency is not inside the event pair
            fn()
            if i >= 2:
                ts.append(lib.tk_last_kernel_ms())
        return float(np.median(ts))

    def rel_err(got, exp):
        got, exp = np.asarray(got, dtype=np.float64), np.asarray(exp, dtype=np.float64)
        nz = exp != 0
        if not np.array_equal(got[~nz], exp[~nz]):
            return float("inf")
        return float(np.max(np.abs(got[nz] - exp[nz]) / np.abs(exp[nz]))) if nz.any() else 0.0

    # the cold-read floor of each small config's byte count under the identical flush: a read-only
    # stream kernel with dot's access pattern (tk_read_floor_f64_device)
    floor_buf = torch.rand(134_283_264 // 8 + 2, dtype=torch.float64, device="cuda")
    sink = torch.empty(148 * 8, dtype=torch.float64, device="cuda")
    res["floor"] = {}
    for name, nbytes in (("cfg1_16MB", 16_000_000), ("cfg3_47MB", 47_199_160), ("cfg2_134MB", 134_283_264)):
        n = nbytes // 8 // 2 * 2
        fms = kernel_ms(lambda: _lib.check(lib.tk_read_floor_f64_device(floor_buf.data_ptr(), n, sink.data_ptr(),
                                                                         int(torch.cuda.current_stream().cuda_stream))))
        res["floor"][name] = {"kernel_ms": fms, "GBps": nbytes / fms / 1e6}
    del floor_buf, sink
    ops = synth.host_operands(1)
    x, y = torch.from_numpy(ops["x"]).cuda(), torch.from_numpy(ops["y"]).cuda()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    ms = kernel_ms(lambda: dv.dot(x, y, out))
    res["cfg1_dot"] = {"kernel_ms": ms, "GBps": 16e6 / ms / 1e6, "bytes": 16_000_000}
    if ck is not None:
        res["cfg1_dot"]["parity"] = {"max_rel_err": rel_err([out.item()], [ck.dot(ops["x"], ops["y"])]),
                                     "tol": 1e-12, "checked_against": "reference"}
    ops = synth.host_operands(2)
    a, xv = torch.from_numpy(ops["a"]).cuda(), torch.from_numpy(ops["x"]).cuda()
    yv = torch.empty(4096, dtype=torch.float64, device="cuda")
    ms = kernel_ms(lambda: dv.matvec(a, xv, yv))
    b = 8 * (4096 * 4096 + 4096 + 4096)
    res["cfg2_matvec"] = {"kernel_ms": ms, "GBps": b / ms / 1e6, "bytes": b}
    if ck is not None:
        res["cfg2_matvec"]["parity"] = {"max_rel_err": rel_err(yv.cpu().numpy(), ck.matvec(ops["a"], ops["x"])),
                                        "tol": 1e-12, "checked_against": "reference"}
    ops = synth.host_operands(3)
    t3 = ops["tensor"]
    dt = DeviceCoo.from_host(t3.subs, t3.vals, t3.shape)
    x3 = torch.from_numpy(ops["x"]).cuda()
    o_s = torch.empty((t3.nnz, 2), dtype=torch.int64, device="cuda")
    o_v = torch.empty(t3.nnz, dtype=torch.float64, device="cuda")
    u = [0]

    def run3():
        u[0] = dt.ttv(x3, 2, o_s, o_v)[0]
    ms = kernel_ms(run3)
    b = t3.nnz * 32 + 8 * 1000 + u[0] * 24
    res["cfg3_ttv"] = {"kernel_ms": ms, "GBps": b / ms / 1e6, "nnz_per_s": t3.nnz / ms * 1e3, "bytes": b, "u": u[0]}
    if ck is not None:
        es, ev, _ = ck.ttv_raw(t3.subs, t3.vals, t3.shape, ops["x"], 2)
        res["cfg3_ttv"]["parity"] = {
            "bit_exact": bool(np.array_equal(es, o_s[:u[0]].cpu().numpy())
                              and np.array_equal(ev.view(np.int64), o_v[:u[0]].cpu().numpy().view(np.int64))),
            "u": int(len(ev)), "checked_against": "reference"}
    del dt, o_s, o_v
    c4 = CFG4
    t4 = DeviceCoo.generate(c4["shape"], c4["nnz"], seed=c4["seed"])
    vecs = {m: uniform_vector(c4["shape"][m], 40 + m) for m in (1, 2, 3)}
    out4 = torch.empty(c4["shape"][0], dtype=torch.float64, device="cuda")
    ms = kernel_ms(lambda: t4.ttv_dense(vecs, 0, out4))
    b = c4["nnz"] * 40 + 3 * 8 * 20000 + 8 * 20000
    res["cfg4_ttv_dense"] = {"kernel_ms": ms, "GBps": b / ms / 1e6, "nnz_per_s": c4["nnz"] / ms * 1e3, "bytes": b}
    if with_cpu:
        # full-size parity: the chain of the reference's ttv_raw (modes 3, 2, 1) on every host
        # thread (keep-mode shards), densified -- the SURVEY 8c config-4 oracle; its time is the
        # config-4 CPU baseline
        s4, v4 = host_tensor(t4)
        vh = {m: vecs[m].cpu().numpy() for m in vecs}
        ref4, el4, kind4 = oracle.ttv_multi_dense_threads(s4, v4, c4["shape"], vh, 0, threads)
        res["cfg4_ttv_dense"]["parity"] = {"rows": int(c4["nnz"]), "max_rel_err": rel_err(out4.cpu().numpy(), ref4),
                                           "tol": 1e-12, "checked_against": kind4 + " (chained ttv_raw)"}
        res["cfg4_ttv_dense"]["cpu_baseline"] = {"value": c4["nnz"] / el4, "unit": "nnz/s", "cores": threads,
                                                 "kind": kind4, "seconds": el4,
                                                 "sample": "full tensor, chained ttv_raw on key-aligned shards"}
        del s4, v4
    # extension (not a BASELINE config): MTTKRP of the config-4 tensor, mode 0,
    # rank 16; bytes = the stream + factor matrices + output (the R-wide gathers hit L2)
    R = 16
    gen = torch.Generator(device="cuda").manual_seed(16)
    fac = {m: torch.rand((c4["shape"][m], R), dtype=torch.float64, device="cuda", generator=gen) for m in (1, 2, 3)}
    out_m = torch.empty((c4["shape"][0], R), dtype=torch.float64, device="cuda")
    ms = kernel_ms(lambda: t4.mttkrp(fac, 0, out_m))
    b = c4["nnz"] * 40 + 4 * 8 * 20000 * R
    res["ext_mttkrp_cfg4_r16"] = {"kernel_ms": ms, "GBps": b / ms / 1e6, "nnz_per_s": c4["nnz"] / ms * 1e3,
                                  "bytes": b, "gathered_GBps": c4["nnz"] * 3 * R * 8 / ms / 1e6}
    del fac, out_m
    del t4
    torch.cuda.empty_cache()
    # the paper's own protocol contracts the middle mode: config-5 tensor, k = 1,
    # the general path (device stable radix sort of (linearised kept key, w), then the same fold);
    # whole call timed by CUDA events (several kernels); inputs 12.8 GB > L2
    c5 = CFG5
    t5 = DeviceCoo.generate(c5["shape"], c5["nnz"], zipf_s=c5["zipf_s"], normal_vals=True, seed=c5["seed"])
    x5 = uniform_vector(c5["shape"][1], c5["xseed"] + 1)
    o_s5 = torch.empty((t5.nnz, 2), dtype=torch.int64, device="cuda")
    o_v5 = torch.empty(t5.nnz, dtype=torch.float64, device="cuda")
    def time_k1():
        ts, u = [], 0
        l0 = lib.tk_launch_count()
        for i in range(3 + 2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            u = t5.ttv(x5, 1, o_s5, o_v5)[0]
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts)), u, (lib.tk_launch_count() - l0) / 5
    ms, u5, launches = time_k1()  # the segmented path (tk_midmode.cu), no library sort
    b = c5["nnz"] * 32 + 8 * c5["shape"][1] + u5 * 24
    res["cfg5_ttv_mode1_sort_path"] = {"call_ms": ms, "GBps": b / ms / 1e6, "nnz_per_s": c5["nnz"] / ms * 1e3,
                                       "bytes": b, "u": u5, "launches_per_call": launches,
                                       "path": "per leading value: in-order accumulation by the suffix key (warp / CTA "
                                               "accumulators; the largest segments by a stable owner-list scatter + "
                                               "serial bucket folds), tk_midmode.cu"}
    keep = (o_s5[:u5].clone(), o_v5[:u5].clone())
    os.environ["TK_MID_MODE"] = "0"  # the previous path, for comparison: CUB stable radix sort per interval
    try:
        ms0, u0, launches0 = time_k1()
    finally:
        os.environ.pop("TK_MID_MODE", None)
    same = bool(u0 == u5 and torch.equal(keep[0], o_s5[:u0]) and torch.equal(keep[1].view(torch.int64), o_v5[:u0].view(torch.int64)))
    res["cfg5_ttv_mode1_sort_path"]["bit_identical_to_cub_split_path"] = same
    del keep
    res["cfg5_ttv_mode1_cub_split_path"] = {"call_ms": ms0, "GBps": b / ms0 / 1e6, "launches_per_call": launches0,
                                            "path": "interval split + cub::DeviceRadixSort (TK_MID_MODE=0)"}
    del t5, o_s5, o_v5
    torch.cuda.empty_cache()
    return res


def multi_dense_measurement(rank, world, steps, warmup, comm):
    """Config 4 sharded across the ranks: the kernel-store merge
    (multi.PeerDenseMerge: every shard's dense-TTV kernel stores its owned keep-mode range into
    all ranks' NVLink-mapped output vectors, then a one-element barrier) against the NCCL
    all-reduce merge of zero-padded partials.  Device time per step (CUDA events, max over
    ranks); the two merged vectors must be bit-identical.  Requires an initialised process group."""
    import torch
    import torch.distributed as dist
    from paper_2510_01495_b200 import multi
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    c4 = CFG4
    shape = c4["shape"]
    full = DeviceCoo.generate(shape, c4["nnz"], seed=c4["seed"])
    vecs = {m: uniform_vector(shape[m], 40 + m) for m in (1, 2, 3)}
    bounds = multi.shard_bounds(full.cols[0], world)
    klo, khi = multi.owned_key_range(full.cols[0], bounds, rank, shape[0])
    t = full.slice(bounds[rank], bounds[rank + 1]) if world > 1 else full
    del full
    torch.cuda.empty_cache()
    merge = multi.PeerDenseMerge(shape[0], torch.cuda.current_device(), comm)
    red = torch.empty(shape[0], dtype=torch.float64, device="cuda")

    def peer_step():
        merge.run(t, vecs, 0, klo, khi)

    def nccl_step():
        t.ttv_dense(vecs, 0, red)
        multi.merge_dense(comm, red)

    res = {}
    for name, fn in (("kernel_store_merge", peer_step), ("nccl_allreduce_merge", nccl_step)):
        for _ in range(warmup):
            fn()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
        res[name] = {"ms_per_step": ms, "nnz_per_s": c4["nnz"] / (ms / 1e3)}
    res["identical"] = bool(torch.equal(merge.out, red))
    res["workload"] = "cfg4_ttv_dense_20000^4_nnz1e8_keep0"
    res["shard_rows"] = t.nnz
    merge.close()
    return res


def run_ours(args):
    import torch
    from paper_2510_01495_b200 import _lib, multi
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    rank, world, local = dist_setup(args)
    lib = _lib.load()
    cfg = dict(CFG5)
    nnz_total = args.nnz or cfg["nnz"]
    shape, k = cfg["shape"], cfg["k"]
    ncpu, threads = cpu_info()

    # ---- operands (outside the timed region) ----
    t_gen = time.perf_counter()
    full = DeviceCoo.generate(shape, nnz_total, zipf_s=cfg["zipf_s"], normal_vals=True, seed=cfg["seed"])
    gen_s = time.perf_counter() - t_gen
    x = uniform_vector(shape[k], cfg["xseed"])
    key = multi.kept_prefix_key(full.cols, 2, shape)
    bounds = multi.shard_bounds(key, world)
    del key
    lo, hi = bounds[rank], bounds[rank + 1]
    t = full.slice(lo, hi, copy=True) if world > 1 else full
    if world > 1:
        del full
    torch.cuda.empty_cache()
    n_local = t.nnz
    out_subs = torch.empty((max(n_local, 1), 2), dtype=torch.int64, device="cuda")
    out_vals = torch.empty(max(n_local, 1), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    comm = make_comm(rank, world)
    pending = [None]  # N > 1: the previous step's count all-gather, finished while this step's kernel runs

    def step():
        u, _, _ = t.ttv(x, k, out_subs, out_vals)
        if world > 1:
            h = comm.counts_start(u, stream)  # NCCL all-gather on the comm's stream, after the TTV
            counts = comm.counts_wait(pending[0]) if pending[0] is not None else None
            pending[0] = h
            return u, counts
        return u, [u]

    def drain():  # the last step's offsets (inside the timed region)
        if pending[0] is None:
            return None
        c = comm.counts_wait(pending[0])
        pending[0] = None
        return c

    for _ in range(args.warmup):
        u_local, counts = step()
    counts = drain() or counts
    torch.cuda.synchronize()

    # ---- timed region ----
    kms = []
    launches0 = lib.tk_launch_count()
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            u_local, counts = step()
            kms.append(lib.tk_last_kernel_ms())
        counts = drain() or counts
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    launches = lib.tk_launch_count() - launches0
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local, world)
    u_total = sum(counts)
    value = nnz_total / (ms / 1e3)

    # roofline of the dominant kernel (the streaming TTV), per launch, this rank's shard
    kern_ms = float(np.mean(kms))
    alg_bytes = n_local * 32 + 8 * shape[k] + u_local * 24
    peak, peak_kind = peaks()
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        if tj.get("nnz") == n_local and tj.get("kernel", "").startswith("ttv_tile_kernel"):
            traffic = tj.get("dram_bytes_per_launch")

    # ---- host copies of the tensor and of the GPU result (outside every timed region) ----
    need_host = (world == 1 and not (args.no_cpu and args.no_e2e)) or (world > 1 and not args.no_e2e)
    subs_h = vals_h = None
    if need_host:
        subs_h, vals_h = host_tensor(t)
    xh = x.cpu().numpy()
    gpu_subs = out_subs[:u_local].cpu().numpy()
    gpu_vals = out_vals[:u_local].cpu().numpy()
    result = digest(gpu_subs, gpu_vals) if rank == 0 and world == 1 else None
    if world == 1:
        del out_subs, out_vals
        torch.cuda.empty_cache()

    # ---- e2e through the drop-in API: kernels().ttv_raw on the pageable numpy arrays a reference
    #      caller holds (H2D of the tensor, TTV, D2H of the result, host reassembly) ----
    e2e = None
    if not args.no_e2e and subs_h is not None:
        e2e = run_e2e(subs_h, vals_h, shape, xh, k, args, gpu_subs, gpu_vals, world, nnz_total)

    parity = None
    cpu_leg = None
    if rank == 0 and world == 1 and not args.no_cpu:
        parity = parity_cfg5(subs_h, vals_h, shape, xh, k, gpu_subs, gpu_vals, threads)
        cpu_leg = {"value": nnz_total / parity["seconds"], "unit": "nnz/s", "cores": threads,
                   "kind": parity["checked_against"],
                   "sample": f"the full config-5 tensor ({nnz_total} rows, same_config): {threads} key-aligned "
                             f"shards on {threads} threads, the reference's ttv_raw(..., release_gil=True) each",
                   "host_cpus": ncpu, "affinity": threads, "seconds": parity["seconds"]}

    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary:
        del subs_h, vals_h, gpu_subs, gpu_vals, t, full
        torch.cuda.empty_cache()
        secondary = secondary_measurements(rank, max(3, min(args.steps, 10)), threads, not args.no_cpu)
        if not args.no_cpu:
            secondary["harness"] = harness_baselines(threads)

    multi_dense = None
    if world > 1 and not args.no_secondary:
        del out_subs, out_vals, t
        torch.cuda.empty_cache()
        multi_dense = multi_dense_measurement(rank, world, max(3, min(args.steps, 10)), 3, comm)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated, seeded; Zipf(1.2) coords, N(0,1) vals)",
            "config": {"workload": WORKLOAD, "nnz": nnz_total, "shape": list(shape), "mode": k, "u": u_total,
                       "parallelism": f"nnz-shard{world}", "l2": "inputs (12.8 GB) larger than L2; no flush",
                       "gen_seconds": round(gen_s, 2)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "frac_vs_nominal_8000": achieved / 8000.0,
                         "kernel": "ttv_tile_kernel<Raw,2,768,32>", "kernel_ms": kern_ms,
                         "alg_bytes_per_launch": alg_bytes},
            "clocks": clocks.summary(),
            "gpu_launches": int(launches),
            "e2e": e2e,
            "cpu_baseline": cpu_leg,
            "parity": parity,
            "result": result,
            "secondary": secondary,
        }
        if multi_dense is not None:
            line["multi_dense"] = multi_dense
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        comm.close()
        dist.destroy_process_group()
    return 0


def run_e2e(subs_h, vals_h, shape, xh, k, args, gpu_subs, gpu_vals, world=1, nnz_total=None):
    """The reference caller's call: ``kernels().ttv_raw(subs, vals, shape, x, k)`` with the
    pageable, read-only numpy arrays a SparseCooTensor holds (pkg/src/tenkern/sparse.py:101-107),
    timed from the host (copies in and out, GPU work and the fresh output arrays inside)."""
    import paper_2510_01495_b200 as tk
    from paper_2510_01495_b200 import _lib
    K = tk.kernels()
    subs_h.flags.writeable = False
    vals_h.flags.writeable = False
    res = K.ttv_raw(subs_h, vals_h, shape, xh, k)
    same = bool(np.array_equal(res[0], gpu_subs) and np.array_equal(res[1].view(np.int64), gpu_vals.view(np.int64)))
    del res
    steps = max(1, min(args.e2e_steps, args.steps))
    ts, native = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        res = K.ttv_raw(subs_h, vals_h, shape, xh, k)
        ts.append(time.perf_counter() - t0)
        native.append(_lib.load().tk_last_call_seconds())
        u = len(res[1])
        del res
    el = max_over_ranks(float(np.mean(ts)), world)  # N > 1: every rank's drop-in call on its shard
    n = subs_h.shape[0] if world == 1 else int(nnz_total)
    return {"value": n / el, "unit": "nnz/s", "h2d_bytes_per_step": int(n * 32 + 8 * xh.shape[0]),
            "h2d_wire_bytes_per_step": int(n * 16 + 8 * xh.shape[0]),  # packed rows (RowPack) + values
            "d2h_bytes_per_step": int(u * 24), "ms_per_step": el * 1e3, "native_ms_per_step": 1e3 * float(np.mean(native)),
            "ms_steps": [round(v * 1e3, 1) for v in ts],
            "steps": steps, "result_matches_device_path": same,
            "path": "kernels().ttv_raw(subs, vals, shape, x, k) on pageable read-only numpy arrays "
                    "(the reference's kernel-module call) -> tk_ttv_f64_host: rows packed to 64-bit words by "
                    "the host thread pool into pinned staging, 8M-row chunks, H2D / TTV / D2H overlapped"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nnz", type=int, default=0, help="override config-5 nnz (debug only)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args)
    if world > 1 and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.gpus > 1 and world == 1:
        return launch_ranks(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
