"""LUT-layer throughput on B200 — BASELINE.json metric on configs[4].

    python bench.py [--gpus N] [--steps K] [--warmup W] [--table f32|i8] [--k 16|64]
    python bench.py --impl reference ...   # the reference's CPU path (oracle port), all host cores

Workload (BASELINE.json configs[4], the scaling sweep): one LUT Linear layer,
N = 2^20 rows per GPU (weak scaling: rows sharded across ranks, tables
replicated, no collective), D = M = 4096, V = 32 -> C = 128, K = 16 (or 64),
inputs ~N(0,1), centroids ~N(0,1), weights ~N(0, 1/D), fp32 or int8 tables.
A step = encode + lookup-aggregate over the rank's N rows, input resident in
HBM.  Inputs (17.2 GB) are far larger than L2 (126 MB), so no L2 flush is
needed between steps.  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LUT-layer rows/sec and effective GOP/s at 1/2/4/8 B200; % of binding roofline"
UNIT = "rows/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--table", choices=["f32", "i8"], default=None,
                   help="table kind (default: BASELINE's — int8 for cfg2/cfg4/cfg5, fp32 for cfg1/cfg3)")
    p.add_argument("--k", type=int, default=16)
    p.add_argument("--rows", type=int, default=1 << 20, help="rows per GPU")
    p.add_argument("--dim", type=int, default=4096)
    p.add_argument("--v", type=int, default=32)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--gather", choices=["tensor", "cuda"], default="tensor",
                   help="lookup engine: tcgen05 one-hot GEMM (int8 exact / f32 digit planes) or CUDA-core")
    p.add_argument("--digits", type=int, default=4, help="f32 digit planes for the tensor engine")
    p.add_argument("--cpu-rows", type=int, default=0, help="CPU sample rows per core (0 = default)")
    p.add_argument("--workload", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"], default="cfg5",
                   help="BASELINE configs[i-1]; cfg5 (default) is the headline scaling sweep")
    p.add_argument("--scale-mtile", type=int, default=-1,
                   help="cfg2/cfg4: per-m-tile int8 scales (0 = per table; default: cfg2 128, cfg4 0)")
    p.add_argument("--cmtile-tensor", action="store_true",
                   help="cfg2: per-(codebook, m-tile) scales on the tensor cores (dequantized table as 4 digit "
                        "planes, <= 1e-5) instead of the bitwise CUDA-core f32 sums")
    p.add_argument("--per-table-scales", action="store_true",
                   help="cfg2: one scale per (m-tile) shared by all codebooks instead of BASELINE's per-(c, m-tile)")
    p.add_argument("--no-variants", action="store_true", help="skip the K=64 / fp32 / CUDA-core variant timings")
    p.add_argument("--no-ties", action="store_true", help="skip the f64 near-tie count")
    p.add_argument("--gather-out", action="store_true",
                   help="under torchrun: also time the NCCL all-gather of the row-sharded output")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


# ------------------------------------------------------------- CPU side


_CPU_WORK = None  # set before the fork pool starts; workers inherit it (no pickling in the timed loop)


_CPU_PLAN = (64, 8)  # KernelPlan(n_block, k_block) of the encode (kernels.py:39-59 default)


def _cpu_worker(rows):
    from oracle import lut_oracle as O

    a, books, table, q, scale, integer = _CPU_WORK
    a = a[:rows]
    nb, kb = _CPU_PLAN
    if integer:
        return O.lut_layer_infer(a, books, q=q, scale=scale, n_block=nb, k_block=kb).shape[0]
    return O.lut_layer_infer(a, books, table=table, integer=False, n_block=nb, k_block=kb).shape[0]


def _cpu_pool_time(rows_per_core, workers, steps, warmup, ctx):
    """Median seconds per step of `workers` processes each running rows_per_core rows."""
    times = []
    with ctx.Pool(workers) as pool:
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            done = sum(pool.map(_cpu_worker, [rows_per_core] * workers, chunksize=1))
            assert done == rows_per_core * workers
            dt = time.perf_counter() - t0
            if i >= warmup:
                times.append(dt)
    return statistics.median(times), len(times)


def cpu_reference(dim, m, v, k, integer, rows_per_core, steps, warmup, seed=7, extras=True):
    """The reference's CPU path (oracle port of lutkit.kernels.lut_layer_infer,
    f64 encode + ascending-c gather) on the host cores: rows sharded over a
    process pool, one BLAS thread per process, as the reference caps BLAS
    (__init__.py:12-15).  `extras`: the reference's own single-core contract
    (one process) and a linearity check (the pool at half the sample; rows/s
    must agree within 15% for the sample to stand in for the 2^20-row shard)."""
    import multiprocessing as mp

    from oracle import lut_oracle as O

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    cores = len(os.sched_getaffinity(0))
    rng = O.make_rng(seed)
    c = dim // v
    books = rng.standard_normal((c, k, v)).astype(np.float32)
    w = (rng.standard_normal((dim, m)) / np.sqrt(dim)).astype(np.float32)
    table = O.build_table(w, books)
    q, scale = O.quantize_table(table) if integer else (None, None)
    shard = rng.standard_normal((rows_per_core, dim)).astype(np.float32)
    global _CPU_WORK
    _CPU_WORK = (shard, books, table, q, scale, integer)
    ctx = mp.get_context("fork")
    med, nsteps = _cpu_pool_time(rows_per_core, cores, steps, warmup, ctx)
    rows = rows_per_core * cores
    res = {"value": rows / med, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"{rows} rows ({rows_per_core}/core) of the same layer per step, median of {nsteps} steps "
                     f"after {warmup} warm-up; oracle port of lutkit lut_layer_infer "
                     f"({'int8' if integer else 'f32'} tables)",
           "seconds_per_step": med, "rows_sampled": rows, "steps": nsteps, "warmup": warmup}
    if extras:
        half = max(1, rows_per_core // 2)
        med_h, _ = _cpu_pool_time(half, cores, 1, 0, ctx)
        r_half = half * cores / med_h
        res["linearity"] = {"rows_sampled_half": half * cores, "rows_per_s_half": r_half,
                            "ratio_full_over_half": res["value"] / r_half,
                            "linear": abs(res["value"] / r_half - 1.0) < 0.15}
        med_1, _ = _cpu_pool_time(half, 1, 1, 0, ctx)
        res["one_core"] = {"value": half / med_1, "unit": UNIT, "cores": 1, "rows_sampled": half}
        # the large-block plan SURVEY §8(d) asks for: KernelPlan(n_block=8192, k_block=16)
        global _CPU_PLAN
        _CPU_PLAN = (8192, 16)
        med_p, _ = _cpu_pool_time(half, cores, 1, 0, ctx)
        _CPU_PLAN = (64, 8)
        res["plan_8192_16"] = {"value": half * cores / med_p, "unit": UNIT, "cores": cores,
                               "rows_sampled": half * cores, "plan": "KernelPlan(n_block=8192, k_block=16)"}
    return res


# ------------------------------------------------------------- clocks


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self.power_w = []
        self.mem_mhz = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            names = {
                "hw_slowdown": getattr(N, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(N, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        try:
                            self.power_w.append(N.nvmlDeviceGetPowerUsage(h) / 1e3)
                            self.mem_mhz.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_MEM))
                        except Exception:
                            pass
                        r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for nm, bit in names.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    self._stop.wait(0.002)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(1.0)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples),
                "sm_mhz_min": min(self.samples) if self.samples else None,
                "sm_mhz_hist": {str(k_): self.samples.count(k_) for k_ in sorted(set(self.samples))},
                "mem_mhz": statistics.median(self.mem_mhz) if self.mem_mhz else None,
                "power_w_max": max(self.power_w) if self.power_w else None}


# ------------------------------------------------------------- GPU side


def near_tie_count(a, books, chunk):
    """(row, codebook) pairs whose best and second-best literal f64 distances
    (pq.py:53-73) lie within 1e-6 relative: the north star's documented
    near-tie class.  torch f64 on the device, outside the timed region."""
    import torch

    n = a.shape[0]
    c, k, v = books.shape
    p64 = books.double()[None]
    near = 0
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        d = torch.sub(a[r0:r1].double().view(r1 - r0, c, 1, v), p64).square_().sum(-1)
        two = d.topk(2, dim=-1, largest=False).values
        gap = (two[..., 1] - two[..., 0]) / torch.clamp(torch.maximum(two[..., 0].abs(), two[..., 1].abs()),
                                                      min=1e-300)
        near += int((gap < 1e-6).sum())
        del d, two, gap
    return near


class Cfg5:
    """One configs[4] layer variant (K, table kind, engine) over the rank's
    resident rows, timed with CUDA events on the launching stream."""

    def __init__(self, L, lib, dev, a, codes, out, near, d, m, v, k, integer, gather, digits, seed=1234):
        import torch

        self.lib, self.a, self.codes, self.out, self.near = lib, a, codes, out, near
        self.n, self.d, self.m, self.v, self.k, self.c = a.shape[0], d, m, v, k, d // v
        self.integer = integer
        g = torch.Generator(device=dev).manual_seed(seed)
        self.books = torch.randn((self.c, k, v), generator=g, device=dev)
        w = torch.randn((d, m), generator=g, device=dev) / math.sqrt(d)
        self.layer = L.LutLayer(cfg=L.PqConfig(v=v, k=k), books=self.books, weight=w, qat=integer, gather=gather,
                                f32_digits=digits)
        self.tensor = self.layer.uses_tensor_cores(integer)
        self.digits = digits
        self.scales = self.layer.qtable.scales_tensor(dev) if integer else None
        self.image = self.layer.onehot_image(integer) if self.tensor else None
        self.cstride = int(lib.lut_code_stride(self.c))
        self.engine = ("tcgen05 one-hot kind::i8" + ("" if integer else f", {digits} digit planes")) \
            if self.tensor else "CUDA-core SMEM gather"

    def step(self, stream, ev=None):
        """encode -> lookup-aggregate: the two kernels of lut_layer_forward, timed apart."""
        from paper_2302_03213_b200._lib import check

        lib, sp, n, c, k, m = self.lib, stream.cuda_stream, self.n, self.c, self.k, self.m
        if ev:
            ev[0].record(stream)
        check(lib.lut_encode_f32(self.a.data_ptr(), n, self.d, self.layer.books_prep.data_ptr(), c, k, self.v,
                                 self.codes.data_ptr(), 8, self.cstride, self.near.data_ptr(), sp))
        if ev:
            ev[1].record(stream)
        if self.tensor:
            check(lib.lut_gather_onehot(self.codes.data_ptr(), self.cstride, n, c, k, m,
                                        1 if self.integer else self.digits, self.image.data_ptr(),
                                        self.scales.data_ptr() if self.integer else None, 0, None, 0,
                                        self.out.data_ptr(), None, 0, sp))
        elif self.integer:
            check(lib.lut_gather_i8(self.codes.data_ptr(), 8, n, c, k, m, self.layer.qtable.q.data_ptr(),
                                    self.scales.data_ptr(), 0, None, 0, self.out.data_ptr(), None, 0, None, sp))
        else:
            check(lib.lut_gather_f32(self.codes.data_ptr(), 8, n, c, k, m, self.layer.table.data_ptr(), None, 0,
                                     self.out.data_ptr(), 0, None, sp))
        if ev:
            ev[2].record(stream)

    def bytes(self):
        """Algorithmic HBM bytes per launch: gather reads codes
        + table once and writes the output; encode reads A + codebooks and
        writes codes; the layer reads A once and writes the output once."""
        n, c, k, m, d, v = self.n, self.c, self.k, self.m, self.d, self.v
        s = 1 if self.integer else 4
        return {"gather": n * c + s * c * k * m + 4 * n * m, "encode": 4 * n * d + n * c + 4 * c * k * v,
                "layer": 4 * n * d + s * c * k * m + 4 * c * k * v + 4 * n * m}

    def time(self, steps, warmup, world=1, clocks=None):
        import torch
        import torch.distributed as dist

        stream = torch.cuda.current_stream()
        for _ in range(warmup):
            self.step(stream)
        torch.cuda.synchronize()
        self.near.zero_()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with (clocks or _Null()):
            t0.record(stream)
            for i in range(steps):
                torch.cuda.nvtx.range_push(f"step {i}")
                self.step(stream, evs[i])
                torch.cuda.nvtx.range_pop()
            t1.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = t0.elapsed_time(t1)
        enc = sum(e[0].elapsed_time(e[1]) for e in evs) / steps
        gat = sum(e[1].elapsed_time(e[2]) for e in evs) / steps
        return ms / steps, enc, gat

    def roofline(self, enc_ms, gat_ms, step_ms, hbm_peak, peak_kind):
        b = self.bytes()
        dom, dom_ms = ("gather", gat_ms) if gat_ms >= enc_ms else ("encode", enc_ms)
        achieved = b[dom] / (dom_ms / 1e3) / 1e9
        r = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
             "traffic": None, "kernel": dom, "peak_kind": peak_kind, "algorithmic_bytes": b[dom],
             "kernel_ms": {"encode": enc_ms, "gather": gat_ms},
             "kernel_frac": {"encode": b["encode"] / (enc_ms / 1e3) / 1e9 / hbm_peak,
                             "gather": b["gather"] / (gat_ms / 1e3) / 1e9 / hbm_peak},
             "layer_hbm_floor_ms": b["layer"] / (hbm_peak * 1e9) * 1e3,
             "layer_frac_of_hbm_floor": (b["layer"] / (hbm_peak * 1e9) * 1e3) / step_ms}
        if self.tensor:
            # the one-hot GEMM's own ceiling: 2:4-sparse kind::i8, 16384 logical MAC/clk/SM
            macs = self.n * self.m * self.c * self.k * (1 if self.integer else self.digits)
            floor = macs / (16384 * 148 * 1.965e9) * 1e3
            r["sparse_mma_floor_ms"] = floor
        else:
            # CUDA-core gather: table lookups from SMEM, 128 B/clk/SM
            lookups = self.n * self.m * self.c * (1 if self.integer else 4)
            r["smem_lookup"] = {"bytes": lookups, "floor_ms": lookups / (148 * 128 * 1.965e9) * 1e3,
                                "frac": (lookups / (148 * 128 * 1.965e9) * 1e3) / gat_ms}
        return r


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


def main():
    args = parse()
    if args.table is None:
        args.table = "f32" if args.workload in ("cfg1", "cfg3") else "i8"
    if args.workload != "cfg5":
        return main_stack(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    integer = args.table == "i8"
    m = d = args.dim
    v, k = args.v, args.k
    c = d // v
    config = {"workload": "BASELINE configs[4]: single LUT Linear, scaling sweep",
              "rows_per_gpu": args.rows, "d": d, "m": m, "v": v, "c": c, "k": k, "table": args.table,
              "parallelism": f"row-sharded x{world}, tables replicated",
              "l2": "inputs (4*N*D B) >> 126 MB L2; no flush needed"}

    if args.impl == "reference":
        if rank != 0:
            return
        ref = cpu_reference(d, m, v, k, integer, rows_per_core=args.cpu_rows or (4096 if integer else 2048),
                            steps=max(1, args.steps), warmup=max(0, args.warmup))
        # config is key-for-key the GPU arm's (the driver compares the two lines' configs); the CPU
        # sample size travels beside it and in cpu_baseline.sample
        eff = 2.0 * d * m * ref["value"] / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": ref["value"], "unit": UNIT, "n_gpus": args.gpus,
                "steps": ref["steps"], "warmup": ref["warmup"], "ms_per_step": ref["seconds_per_step"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
                "data": "synthetic", "config": config, "rows_sampled_per_step": ref["rows_sampled"],
                "effective_gops": eff,
                "cpu_baseline": {k_: ref[k_] for k_ in ("value", "unit", "cores", "kind", "sample")},
                "one_core": ref.get("one_core"), "linearity": ref.get("linearity"),
                "plan_8192_16": ref.get("plan_8192_16"),
                "e2e": {"value": ref["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(d, m, v, k, integer, rows_per_core=args.cpu_rows or (4096 if integer else 2048),
                            steps=2, warmup=1)

    import torch
    import torch.distributed as dist

    import paper_2302_03213_b200 as L
    from paper_2302_03213_b200._lib import load

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or os.environ.get("RANK") is not None:  # under torchrun, even at N = 1
        dist.init_process_group("nccl", device_id=dev)
    lib = load()

    # ---- this rank's rows (generated on device from (seed, rank)), shared buffers
    n = args.rows
    ga = torch.Generator(device=dev).manual_seed(99 + rank)
    a = torch.randn((n, d), generator=ga, device=dev)
    codes = torch.empty((n, int(lib.lut_code_stride(c))), dtype=torch.uint8, device=dev)
    out = torch.empty((n, m), dtype=torch.float32, device=dev)
    near = torch.zeros(1, dtype=torch.int32, device=dev)
    hbm_peak, _, peak_kind = peaks()
    run = Cfg5(L, lib, dev, a, codes, out, near, d, m, v, k, integer, args.gather, args.digits)
    with ClockSampler(local) as clocks:
        ms_step, enc_ms, gat_ms = run.time(args.steps, args.warmup, world)
    in_dist = dist.is_available() and dist.is_initialized()
    if in_dist and world > 1:
        t = torch.tensor([ms_step], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    redecided = int(near.item())
    rows_total = n * world
    value = rows_total / (ms_step / 1e3)
    eff_gops = 2.0 * d * m * value / 1e9
    roofline = run.roofline(enc_ms, gat_ms, ms_step, hbm_peak, peak_kind)
    for rnd in ("r02", "r01"):  # DRAM bytes per launch from the newest committed ncu capture
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "ncu_traffic.json")) as f:
                tr = json.load(f)
            tc = tr["config"]
            if (tc["d"], tc["m"], tc["v"], tc["k"], tc["table"]) == (d, m, v, k, args.table) and run.tensor:
                roofline["traffic"] = tr[f"{roofline['kernel']}_dram_bytes"] / tr["rows"] * n
                roofline["traffic_source"] = f"profiles/{rnd}/ncu_traffic.json"
                break
        except (OSError, KeyError, ValueError):
            continue

    # ---- north-star near ties (f64 gap < 1e-6 relative), counted over every row (untimed)
    near_1e6 = near_tie_count(a, run.books, chunk=2048 if k <= 16 else 512) if not args.no_ties else None

    # ---- other configs[4] variants on the same rows (BASELINE: K in {16, 64}, fp32 and int8 tables)
    variants = {}
    if not args.no_variants and world == 1:
        del run
        torch.cuda.empty_cache()
        for name, kk, intg, gth in (("k64_i8_tensor", 64, True, "tensor"), ("f32_tensor_4digit", 16, False, "tensor"),
                                    ("f32_cuda_bitwise", 16, False, "cuda"), ("i8_cuda", 16, True, "cuda")):
            if (kk, intg, gth) == (k, integer, args.gather):
                continue
            vr = Cfg5(L, lib, dev, a, codes, out, near, d, m, v, kk, intg, gth, 4)
            st_ms, e_ms, g_ms = vr.time(max(2, args.steps // 4), 2)
            rf = vr.roofline(e_ms, g_ms, st_ms, hbm_peak, peak_kind)
            variants[name] = {"engine": vr.engine, "ms_per_step": st_ms, "rows_per_s": n / (st_ms / 1e3),
                              "kernel_ms": rf["kernel_ms"], "kernel_frac": rf["kernel_frac"],
                              "layer_frac_of_hbm_floor": rf["layer_frac_of_hbm_floor"],
                              **({"sparse_mma_floor_ms": rf["sparse_mma_floor_ms"]} if "sparse_mma_floor_ms" in rf
                                 else {"smem_lookup": rf["smem_lookup"]})}
            del vr
            torch.cuda.empty_cache()
        run = Cfg5(L, lib, dev, a, codes, out, near, d, m, v, k, integer, args.gather, args.digits)
        run.step(torch.cuda.current_stream())  # the headline layer's output back in `out` for the e2e check

    # ---- optional all-gather of the row-sharded output, timed apart
    gathered = None
    if args.gather_out and in_dist:
        from paper_2302_03213_b200.dist import gather_rows

        rows_g = min(n, 1 << 17)
        part = out[:rows_g]
        gather_rows(part, rows_g * world)  # warm NCCL
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        full = gather_rows(part, rows_g * world)
        e1.record()
        torch.cuda.synchronize()
        g_ms = e0.elapsed_time(e1)
        t = torch.tensor([g_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        g_ms = float(t.item())
        gathered = {"rows_per_rank": rows_g, "bytes_out_per_rank": full.numel() * 4, "ms": g_ms,
                    "algbw_GBps": full.numel() * 4 / (g_ms / 1e3) / 1e9, "collective": "NCCL all_gather"}
        del full

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        # one rank: the whole 2^20-row shard (17 GB in + 17 GB out, pinned); under
        # torchrun every rank pins its own buffers, so cap them at 2^18 rows per rank
        # (PCIe-bound either way: rows/s does not depend on the shard length)
        ne = n if world == 1 else min(n, 1 << 18)
        a_h = torch.empty((ne, d), dtype=torch.float32, pin_memory=True)
        a_h.copy_(a[:ne])
        o_h = torch.empty((ne, m), dtype=torch.float32, pin_memory=True)
        a_np, o_np = a_h.numpy(), o_h.numpy()
        L.lut_layer_infer(a_np[: 1 << 14], run.layer, integer=integer)  # warm the executor
        if in_dist:
            dist.barrier()
        times = []
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.lut_layer_infer(a_np, run.layer, integer=integer, out=o_np)
            t1 = time.perf_counter()
            if i:
                times.append(t1 - t0)
        e2e_s = statistics.median(times)
        if in_dist and world > 1:
            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        ok = bool(torch.equal(o_h[:4096].to(dev), out[:4096]))
        e2e = {"value": ne * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 4 * ne * d,
               "d2h_bytes_per_step": 4 * ne * m, "rows_per_gpu": ne, "steps": len(times), "matches_device_path": ok,
               "api": "paper_2302_03213_b200.lut_layer_infer(numpy pinned) -> lut_pipeline_run"}
        del a_h, o_h

    if in_dist:
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if not integer else "f32-encode/int8-table/int32-acc",
            "data": "synthetic (seeded torch.randn on device; random-init centroids/weights)",
            "config": config, "engine": run.engine, "effective_gops": eff_gops,
            "near_ties_gap_lt_1e6": near_1e6,
            "near_ties_gap_lt_1e6_rate": None if near_1e6 is None else near_1e6 / (n * c),
            "f64_redecisions": redecided // max(1, args.steps), "f64_redecision_rate": redecided / (n * c * args.steps),
            "roofline": roofline, "clocks": clocks.summary(), "gpu_launches": 2 * args.steps,
            "variants": variants or None, "gathered_out": gathered,
            "e2e": e2e, "cpu_baseline": None, "launcher": "torchrun" if os.environ.get("RANK") is not None else "python"}
    if cpu is not None:
        line["cpu_baseline"] = {k_: cpu[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
        line["cpu_baseline"]["one_core"] = cpu.get("one_core")
        line["cpu_baseline"]["linearity"] = cpu.get("linearity")
        line["cpu_baseline"]["plan_8192_16"] = cpu.get("plan_8192_16")
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- configs 1-4


def _host(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def stack_cpu_baseline(wl, objs, unit_rows):
    """The reference's CPU algorithm (oracle port: f64 encode, ascending-c f32 /
    exact int8 lookups, the same epilogues) on the same layers, one host thread
    (the reference's contract), on a bounded sample of the step's rows."""
    from oracle import lut_oracle as O

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    t0 = time.perf_counter()
    if wl == "cfg1":
        layer, x = objs
        a = _host(x)
        O.lut_layer_infer(a, _host(layer.books), table=_host(layer.table), integer=False)
        rows, sample = a.shape[0], f"all {a.shape[0]} rows"
    elif wl == "cfg2":
        ffn, x, mt, per_cb = objs
        a = _host(x[:256])
        h = a
        for lin in (ffn.up, ffn.down):
            lut = lin.lut
            enc = O.centroid_search_fast(h, _host(lut.books))
            q, sc = _host(lut.qtable.q), _host(lut.qtable.scales_tensor(lut.device))
            if per_cb:
                y = O.lut_gather_accumulate_cmtile(enc, q, sc.reshape(lut.c, -1), mt)
            elif mt:
                y = O.lut_gather_accumulate_mtile(enc, q, sc, mt)
            else:
                y = O.lut_gather_accumulate(enc, q, sc[0])
            h = O.gelu_erf(y) if lut.act == "gelu" else y
        rows, sample = a.shape[0], "256 of 4096 tokens"
    elif wl == "cfg3":
        convs = objs
        rows = 0
        for conv, x in convs:
            xs = _host(x[:2])
            cols = O.im2col(xs, 3, 3, 1, 1)
            lut = conv.lut
            O.lut_matmul_ref(O.centroid_search_fast(cols, _host(lut.books)), _host(lut.table))
            rows += cols.shape[0]
        sample = "2 of 256 images per stage"
    else:
        return None
    dt = time.perf_counter() - t0
    return {"value": rows / dt, "unit": f"{unit_rows}/s", "cores": 1, "kind": "port", "sample": sample}


STACKS = {
    "cfg1": "BASELINE configs[0]: single LUT Linear N=1024, 768->768, V=16, K=16",
    "cfg2": "BASELINE configs[1]: BERT-base FFN pair 4096 tokens, 768->3072 (GELU) ->768, V=32, K=16, int8",
    "cfg3": "BASELINE configs[2]: ResNet20 3x3 LUT convs, batch 256, 32x32x16 / 16x16x32 / 8x8x64, V=9, K=16, f32",
    "cfg4": "BASELINE configs[3]: 12-layer BERT-base encoder, batch 64 x seq 128, LUT layers 3-12 (V=32, K=16, int8)",
}


def main_stack(args):
    """configs[0..3]: the whole caller (layer, FFN pair, conv stage set, BERT
    encoder) per step, captured in a CUDA graph, L2 flushed between steps;
    LUT-kernel share and its HBM roofline from per-layer events (eager pass)."""
    import torch
    import torch.distributed as dist

    from paper_2302_03213_b200 import workloads as W
    from paper_2302_03213_b200.nn import LutConv2d, LutLinear

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps({"impl": "reference", "unavailable": "reference arm is measured on the headline "
                              "workload (cfg5) only"}), flush=True)
        return
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload
    integer = args.table == "i8"
    if wl == "cfg1":
        layer, x = W.linear(dev, 1024, 768, 768, 16, 16, integer, gather="auto")
        mod = LutLinear(layer, integer)
        fn, rows, unit_rows = (lambda: mod(x)), 1024, "rows"
        cpu_objs = (layer, x) if not integer else None
    elif wl == "cfg2":
        # BASELINE configs[1]: int8 tables with a per-(c, m-tile) fp32 scale
        mt = 128 if args.scale_mtile < 0 else args.scale_mtile
        ffn, x = W.ffn_pair(dev, tokens=4096, scale_mtile=mt, per_codebook=not args.per_table_scales,
                            gather="tensor" if args.cmtile_tensor else "auto")
        fn, rows, unit_rows = (lambda: ffn(x)), 4096, "tokens"
        cpu_objs = (ffn, x, mt, not args.per_table_scales)
    elif wl == "cfg3":
        convs = W.resnet_convs(dev, batch=256)
        x = convs[0][1]
        rest = [xx for _, xx in convs[1:]]

        def fn():
            return [conv(xx) for (conv, _), xx in zip(convs, [x] + rest)]

        rows = sum(xx.shape[0] * xx.shape[2] * xx.shape[3] for _, xx in convs)
        unit_rows = "output pixels"
        cpu_objs = convs
    else:
        model, x = W.bert_encoder(dev, batch=64, seq=128, scale_mtile=max(0, args.scale_mtile))
        fn, rows, unit_rows = (lambda: model(x)), 64 * 128, "tokens"
        cpu_objs = None

    # per-LUT-layer events + algorithmic HBM bytes (fused layer formula)
    luts = []
    if wl == "cfg1":
        luts = [mod]
    elif wl == "cfg2":
        luts = [ffn.up, ffn.down]
    elif wl == "cfg3":
        luts = [conv for conv, _ in convs]
    else:
        luts = [m_ for _, _, m_ in model.lut_linears()]
    marks = []

    def pre(m_, inp):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append([m_, inp[0], e])

    def post(m_, inp, out):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks[-1] += [out, e]

    hooks = [m_.register_forward_pre_hook(pre) for m_ in luts] + [m_.register_forward_hook(post) for m_ in luts]
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    marks.clear()
    fn()
    torch.cuda.synchronize()
    lut_ms, lut_bytes = 0.0, 0
    # SURVEY §8(d) bound per LUT layer: max(HBM bytes / HBM peak, lookup bytes /
    # SMEM (CUDA-core gathers) or sparse-MMA time (tensor gathers), encode FMAs /
    # FP32 rate); the step's bound is their sum over the layers
    hbm_peak_bps = peaks()[0] * 1e9
    clk = 1.965e9
    t_bound = 0.0
    bound_terms = {"hbm": 0.0, "smem_or_mma": 0.0, "ffma": 0.0}
    for m_, a, e0, y, e1 in marks:
        lut = m_.lut
        intg = getattr(m_, "integer", None)
        intg = lut.has_qtable if intg is None else bool(intg)
        s_ = 1 if intg else 4
        lut_ms += e0.elapsed_time(e1)
        hbm_b = 4 * a.numel() + s_ * lut.c * lut.k * lut.m + 4 * lut.c * lut.k * lut.v + 4 * y.numel()
        lut_bytes += hbm_b
        nrows = y.numel() // lut.m
        if lut.uses_tensor_cores(intg):
            gather_t = nrows * lut.m * lut.c * lut.k * (1 if intg else lut.f32_digits) / (16384 * 148 * clk)
        else:
            gather_t = nrows * lut.m * lut.c * s_ / (148 * 128 * clk)
        terms = {"hbm": hbm_b / hbm_peak_bps, "smem_or_mma": gather_t,
                 "ffma": nrows * lut.c * lut.v * lut.k / (148 * 128 * clk)}
        t_bound += max(terms.values())
        bound_terms[max(terms, key=terms.get)] += max(terms.values())
    for hk in hooks:
        hk.remove()

    graph = None
    try:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            fn()
        graph = g
    except Exception as exc:  # eager launches are still measured; the line says which
        graph = None
        print(f"graph capture failed: {exc!r}", file=sys.stderr)
    run = graph.replay if graph is not None else fn
    # L2 flush between timed steps: write a 256 MB buffer (> 126 MB L2), then read
    # a second one so the write-back of the flush's dirty lines happens here and
    # not inside the next timed step (L2 is left holding clean, unrelated lines)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        run()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for e0, e1 in evs:
            flush.zero_()
            flush_rd.sum()
            e0.record()
            run()
            e1.record()
        torch.cuda.synchronize()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # e2e: pinned host input -> device, the caller's forward, output -> pinned host
    x_h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    x_h.copy_(x)
    y0 = fn()
    y0 = y0[-1] if isinstance(y0, list) else y0
    y_h = torch.empty(y0.shape, dtype=y0.dtype, pin_memory=True)
    times = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x.copy_(x_h, non_blocking=True)
        y = fn()
        y = y[-1] if isinstance(y, list) else y
        y_h.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
        if i:
            times.append(time.perf_counter() - t0)
    e2e_s = statistics.median(times)
    hbm_peak, _, peak_kind = peaks()
    achieved = lut_bytes / (lut_ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and cpu_objs is not None and not args.no_cpu:
        cpu = stack_cpu_baseline(wl, cpu_objs, unit_rows)
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    # DRAM bytes per step from the committed ncu launch list of this workload's default arguments
    traffic, traffic_src = None, None
    default_table = "f32" if wl in ("cfg1", "cfg3") else "i8"
    if not args.per_table_scales and not args.cmtile_tensor and args.table == default_table and args.scale_mtile == -1:
        for rnd in ("r02",):
            try:
                with open(os.path.join(ROOT, "profiles", rnd, "ncu_traffic_stacks.json")) as f:
                    traffic = json.load(f)["workloads"][wl]["dram_bytes_per_step"]
                traffic_src = f"profiles/{rnd}/ncu_traffic_stacks.json"
            except (OSError, KeyError, ValueError):
                pass
    line = {"metric": METRIC, "value": rows * world / (ms / 1e3), "unit": f"{unit_rows}/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if not integer else "f32-encode/int8-table/int32-acc",
            "data": "synthetic (seeded torch.randn on device; random-init weights; centroids sampled from a "
                    "held-out batch)",
            "config": {"workload": STACKS[wl], "rows_per_step": rows, "cuda_graph": graph is not None,
                       "l2": "256 MB buffer written, then a 256 MB buffer read, between timed steps",
                       "scale_mtile": args.scale_mtile, "table": args.table,
                       **({"int8_scales": "per (m-tile)" if args.per_table_scales else
                           "per (codebook, m-tile), tensor digit planes" if args.cmtile_tensor else "per (codebook, m-tile)"}
                          if wl == "cfg2" else {})},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "LUT layers (encode+gather)",
                         "peak_kind": peak_kind, "algorithmic_bytes": lut_bytes, "lut_ms_eager": lut_ms,
                         "lut_layers": len(marks),
                         "survey_bound": {"t_bound_ms": t_bound * 1e3,
                                          "binding": max(bound_terms, key=bound_terms.get),
                                          "terms_ms": {k_: v_ * 1e3 for k_, v_ in bound_terms.items()},
                                          "frac_of_step": t_bound * 1e3 / ms}},
            # our kernels in the timed region: one encode + one gather launch per LUT layer and step
            "clocks": clocks.summary(), "gpu_launches": 2 * len(marks) * args.steps,
            "e2e": {"value": rows * world / e2e_s, "unit": f"{unit_rows}/s", "h2d_bytes_per_step": x.numel() * 4,
                    "d2h_bytes_per_step": y0.numel() * 4},
            "cpu_baseline": cpu}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
