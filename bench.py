#!/usr/bin/env python
"""bench.py -- Endor (arXiv 2406.11674) bitmap-sparse decompression on B200.

Metric (BASELINE.json): "Endor decompress dense-GB/s/GPU; offloaded OPT-66B
layer ms at 1-8 B200".  Workload (BASELINE.json configs[1], scaled weakly):
an OPT-66B decoder layer's six f16 weight matrices (q/k/v/out 9216x9216,
fc1 9216x36864, fc2 36864x9216), magnitude-pruned to 50% with the reference's
own synth_weight + magnitude_prune (bit-exact GPU restatements), compressed
to bitmap + packed values.  At N GPUs a step covers N consecutive layers, every
matrix row-block sharded across the N GPUs (north star (c)), so per-GPU work
is one layer's bytes ("scaling": "weak"); no data-path collective.

  value  decompress dense-GB/s, whole job: inputs resident in HBM, one step =
         count + expand for every shard this rank owns; CUDA events on the
         launching stream; max over ranks; inputs (3.2 GB/step/GPU) >> L2.
  e2e    the same metric through the C-ABI offload pipeline over HOST pinned
         buffers: H2D of the compressed shards (copy stream) overlapped with
         decompress + GEMV (compute stream), D2H of every op's y; device-timed.
         Its ms_per_step is the offloaded layer time.
  roofline  the expand kernel (dominant): algorithmic bytes (bitmap n/8 +
         values nnz*2 + dense n*2) / its event-timed duration vs the measured
         HBM copy peak (MEASURED_PEAKS.json).
  cpu_baseline  the reference's own decompress (oracle/_ref, compiled from
         /root/reference) on the host cores, rank 0 at N=1, bounded sample.

--impl reference: the reference's CPU decompress (decompress_chunk_into fanned
over every host core, its documented parallel contract) on one full OPT-66B
layer per step; prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Endor decompress dense-GB/s/GPU; offloaded OPT-66B layer ms at 1-8 B200"
UNIT = "GB/s"
SPARSITY = 0.5
WORKLOAD = "opt-66b decoder layer (q,k,v,out 9216^2; fc1 9216x36864; fc2 36864x9216) f16 @50% unstructured"
PCIE_GEN5_X16_GBS = 63.0


def env_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def numa_pin(gpu: int) -> None:
    """Bind this rank to the CPUs NVML reports as local to its GPU, so pinned
    host buffers (first-touched by this process) sit on the GPU's NUMA node and
    each rank's H2D uses its own socket's memory (north star (c): every GPU
    streams its shards over its own PCIe link)."""
    try:
        import pynvml
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v for v in vis.split(",") if v.strip()]
        phys = int(ids[gpu]) if ids and gpu < len(ids) and ids[gpu].strip().isdigit() else gpu
        pynvml.nvmlInit()
        pynvml.nvmlDeviceSetCpuAffinity(pynvml.nvmlDeviceGetHandleByIndex(phys))
    except Exception:
        pass


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled
    in-process every millisecond (a sub-10 ms region still gets samples), with
    nvidia-smi as the fallback where NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int, period_s: float = 0.001):
        self.idx = gpu_index
        self.period = period_s
        self.samples = []  # (sm_mhz, max_mhz, set(reasons), perf_counter time)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
            phys = int(vis[gpu_index]) if vis and gpu_index < len(vis) and vis[gpu_index].strip().isdigit() \
                else gpu_index
            h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            self._max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))  # ~3 ms per call
            self._nvml = (pynvml, h, bits)
            t = time.perf_counter()
            self._sample()  # first queries are slow (driver-side setup): pay it here
            self.nvml_sample_ms = round((time.perf_counter() - t) * 1e3, 3)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml:
            nv, h, bits = self._nvml
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            return (float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), self._max_mhz,
                    {n for n, bit in zip(self.NAMES, bits) if r & bit}, time.perf_counter())
        out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q,
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        return (float(f[0]), float(f[1]), {n for n, v in zip(self.NAMES, f[2:6]) if v.lower() == "active"},
                time.perf_counter())

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(self.period if self._nvml else 0.2)

    def __enter__(self):
        # the launching thread holds the GIL between its (GIL-releasing) CUDA
        # calls; a short switch interval lets the poller run inside short regions
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(0.0002)
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)
        sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))),
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi",
                "samples_in_timed_region": getattr(self, "in_region", len(self.samples))}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def build_shards(E, catalog, rank, world, dev):
    """This rank's row shards of layers 0..world-1: every whole matrix is
    generated and compressed on the device (bit-exact synth/prune/compress
    kernels), then the rank's shard is SLICED out of the compressed tensor --
    bitmap bits [r0 C, r1 C), values [rank(r0 C), rank(r1 C)) -- into its own
    buffers, as the per-GPU transfer of that slice would deliver it
    (shard.shard_tensor; no re-compression).  Returns a list of dicts."""
    import torch
    from paper_2406_11674_b200 import shard as S
    spec = catalog.model_catalog("opt-66b")
    out = []
    for layer in range(world):
        for oi, op in enumerate(spec.ops):
            sh = S.row_shard(op.rows, op.cols, rank, world)
            w = E.synth_weight(op.rows, op.cols, catalog.op_seed(layer, oi), device=dev)
            E.magnitude_prune(w, SPARSITY, inplace=True)
            t = E.compress(w)
            del w
            if world > 1:
                t = S.shard_tensor(t, sh, copy=True)
            out.append({"name": f"L{layer}.{op.name}[{sh.r0}:{sh.r1}]", "t": t, "rows": sh.rows,
                        "cols": op.cols, "n": sh.rows * op.cols, "nnz": t.nnz()})
        torch.cuda.empty_cache()
    return out


def golden_parity(shards, world, rank=0):
    """CRC-32 of every decompressed layer-0 matrix vs the REFERENCE's decompress
    of the same seeds (tests/golden/large.json).  At N=1 the shards are whole
    matrices; at N>1 every rank checksums its own row shards and rank 0 joins
    them in row order with crc32_combine (the shards never move)."""
    import zlib
    from paper_2406_11674_b200 import shard as S
    p = os.path.join(ROOT, "tests", "golden", "large.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        gold = {g["name"]: g for g in json.load(f)}
    mine = []
    for s in shards:
        name = "opt-66b." + s["name"].split("[")[0]
        if name not in gold:
            continue
        flat = s["out"].data
        c = 0
        for i in range(0, flat.numel(), 256 << 20):
            c = zlib.crc32(flat[i: i + (256 << 20)].cpu().numpy().tobytes(), c)
        r0 = int(s["name"].split("[")[1].split(":")[0])
        mine.append((name, r0, c & 0xFFFFFFFF, int(flat.numel()), int(s["nnz"])))
    parts = [mine]
    if world > 1:
        import torch.distributed as dist
        parts = [None] * world
        dist.all_gather_object(parts, mine)
    if rank != 0:
        return None
    by = {}
    for part in parts:
        for name, r0, c, nbytes, nnz in part:
            by.setdefault(name, []).append((r0, c, nbytes, nnz))
    ok, checked = True, 0
    for name, lst in by.items():
        c, nnz = 0, 0
        for r0, ci, nb, nz in sorted(lst):
            c = S.crc32_combine(c, ci, nb)
            nnz += nz
        ok &= c == gold[name]["crc_dense"] and nnz == gold[name]["nnz"]
        checked += 1
    return {"vs": "reference decompress CRC-32 (tests/golden/large.json)" +
            (f", {world} row shards per matrix joined by crc32_combine" if world > 1 else ""),
            "tensors": checked, "bit_exact": ok}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2406_11674_b200 import _lib, catalog, codec as E
    from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy

    world, rank, local = env_dist()
    # ENDOR_BENCH_SHARE_GPU=1: a code-path check of N>1 on a box with fewer GPUs
    # than ranks (ranks share devices, gloo plumbing; the numbers are not a measurement)
    share = os.environ.get("ENDOR_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa_pin(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()

    shards = build_shards(E, catalog, rank, world, dev)
    nmax = max(s["n"] for s in shards)
    for s in shards:
        s["dense"] = torch.empty(s["n"] * 2 + 16, dtype=torch.uint8, device=dev)
        s["out"] = E.DenseMatrix(s["rows"], s["cols"], E.Dtype.F16, s["dense"][: s["n"] * 2])
    # one batch per step: every weight shard this rank owns (6 per layer, 6 N at N
    # GPUs, <= 64 per launch).  Headline: the reference's parallel API
    # decompress_chunked (codec.hpp:205) with a RankIndex at chunk 1024 built once
    # at load time (like compression, offline): one expand launch per step.  Also
    # reported: decompress (codec.hpp:157), no index (count + expand launches).
    per_layer = len(shards)
    groups = [shards]
    for s in shards:
        s["idx"] = E.build_rank_index(s["t"].bitmap, 1024)
    plans_idx = [E.BatchPlan([s["t"] for s in g], [s["out"] for s in g], indices=[s["idx"] for s in g])
                 for g in groups]
    plans_noidx = [E.BatchPlan([s["t"] for s in g], [s["out"] for s in g]) for g in groups]
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(plans, sample_clocks=False):
        """warmup, then exactly `steps` steps between events on the launching stream;
        barrier + synchronize on both sides; max over ranks."""
        clk = ClockSampler(local) if sample_clocks else None
        if clk:
            clk.__enter__()  # polling from before the warm-up: it is running when the region opens
        for _ in range(args.warmup):
            for p in plans:
                p.launch(sp)
        for p in plans:
            p.sync(sp)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_open = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            for p in plans:
                p.launch(sp)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_close = time.perf_counter()
        if clk:
            clk.in_region = sum(1 for s in list(clk.samples) if t_open <= s[3] <= t_close)
            # a sub-second timed region yields few nvidia-smi samples: keep the same
            # load running (untimed) until at least 3 samples exist
            t_end = time.time() + 3.0
            while len(clk.samples) < 3 and time.time() < t_end:
                for p in plans:
                    p.launch(sp)
                torch.cuda.synchronize()
            clk.__exit__()
        barrier()
        torch.cuda.synchronize()
        for p in plans:
            p.sync(sp)  # any device-detected corruption raises here
        return max_over_ranks(ev0.elapsed_time(ev1)) / args.steps, clk

    dense_rank = sum(s["n"] * 2 for s in shards)
    comp_rank = sum((s["n"] + 7) // 8 + s["nnz"] * 2 for s in shards)
    alg_rank = sum(catalog.algorithmic_bytes(s["n"], s["nnz"]) for s in shards)
    peak, peak_src = measured_peak()

    # ---- device-resident decompress: the `value` -------------------------------------
    ms_noidx, _ = timed(plans_noidx)
    parity_noidx = golden_parity(shards, world, rank)
    ms_step, clk = timed(plans_idx, sample_clocks=True)
    parity = golden_parity(shards, world, rank)
    if parity is not None and parity_noidx is not None:
        parity["bit_exact"] = parity["bit_exact"] and parity_noidx["bit_exact"]
        parity["paths"] = "decompress_chunked(idx 1024) and decompress"
    value = world * dense_rank / (ms_step * 1e-3) / 1e9
    launches = len(plans_idx) * args.steps
    no_index = {"api": "decompress (codec.hpp:157): count + expand launch per layer",
                "value": round(world * dense_rank / (ms_noidx * 1e-3) / 1e9, 2),
                "ms_per_step": round(ms_noidx, 4),
                "step_frac": round(alg_rank / (ms_noidx * 1e-3) / 1e9 / peak, 4)}

    # ---- instrumented pass: per-kernel durations (roofline) --------------------------
    # events bracket each launch on the launching stream; one expand launch covers
    # a layer's six shards, so its algorithmic bytes are the layer's
    def kernel_times(plans, with_count):
        count_ms, expand_ms, alg, evs = 0.0, 0.0, 0, []
        for _ in range(args.steps):
            for p in plans:
                a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                a.record(stream)
                if with_count:
                    p.launch(sp, phase=1)
                b.record(stream)
                p.launch(sp, phase=2)
                c.record(stream)
                evs.append((a, b, c, p))
        torch.cuda.synchronize()
        for a, b, c, p in evs:
            count_ms += a.elapsed_time(b) if with_count else 0.0
            expand_ms += b.elapsed_time(c)
            alg += sum(catalog.algorithmic_bytes(t.element_count(), t.nnz()) for t in p.tensors)
        return count_ms / len(evs), expand_ms / len(evs), alg // len(evs)

    _, expand_ms, expand_alg = kernel_times(plans_idx, False)
    count_ms, _, _ = kernel_times(plans_noidx, True)
    achieved = expand_alg / (expand_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "bench_expand_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    mix_ceiling = None  # streaming ceiling for this read/write mix (profiles/r01/mix_ceiling.txt)
    mp = os.path.join(ROOT, "profiles", "bench_expand_traffic.json")
    if os.path.exists(mp):
        with open(mp) as f:
            mix_ceiling = json.load(f).get("mix_ceiling_gbs")
    roofline = {"bound": "hbm", "kernel": "expand_tma_kernel<2, 0, 0, 1>", "achieved": round(achieved, 1),
                "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": "recorded ncu --set full capture of this kernel on this build "
                                  "(profiles/bench_expand_traffic.json), not measured in this run",
                "alg_bytes_per_launch": expand_alg,
                "avg_launch_us": round(expand_ms * 1e3, 2),
                "count_kernel_avg_us_no_index_path": round(count_ms * 1e3, 2),
                "mix_ceiling_gbs": mix_ceiling,
                "frac_of_mix_ceiling": round(achieved / mix_ceiling, 4) if mix_ceiling else None,
                "frac_of_spec_8000gbs": round(achieved / 8000.0, 4),  # also vs the 8 TB/s spec
                "step_frac": round(alg_rank / (ms_step * 1e-3) / 1e9 / peak, 4)}

    # ---- e2e: offload pipeline over pinned host buffers ----------------------------------
    e2e = None
    if not args.no_e2e:
        g = torch.Generator(device="cpu").manual_seed(1234 + rank)
        hops = []
        for s in shards:
            t = s["t"]
            x = ((torch.rand(s["cols"], generator=g) * 2 - 1).half()).to(dev)
            hops.append(HostOp(s["rows"], s["cols"], 0, pinned_copy(t.bitmap.data), pinned_copy(t.values),
                               s["nnz"], x=x, y=torch.empty(s["rows"], dtype=torch.float32, device=dev),
                               y_host=torch.empty(s["rows"], dtype=torch.float32, pin_memory=True)))
        pipe = OffloadPipeline(local, nmax, ring_depth=2)
        for _ in range(max(1, args.warmup)):
            pipe.run(hops, sync=True)
        # GEMV parity on the pipeline's output vs an fp32 reference of the same W
        ref_dense = shards[-1]["dense"][: shards[-1]["n"] * 2].view(torch.float16).reshape(shards[-1]["rows"], -1)
        E.decompress(shards[-1]["t"], out=E.DenseMatrix(shards[-1]["rows"], shards[-1]["cols"], E.Dtype.F16,
                                                        shards[-1]["dense"][: shards[-1]["n"] * 2]))
        gemv_err = gemv_errors(hops[-1].y_host, ref_dense, hops[-1].x)
        torch.cuda.synchronize()
        barrier()
        ops_all = hops * args.steps
        with ClockSampler(local, float(os.environ.get("ENDOR_E2E_POLL_S", "0.02"))) as clk2:
            pipe.run(ops_all, sync=True)
        st = pipe.stats()
        barrier()
        # the same ops with W materialised (decompress, then dense GEMV), for contrast
        mops = [HostOp(h.rows, h.cols, 0, h.bitmap, h.values, h.nnz, x=h.x, y=h.y, y_host=h.y_host,
                       materialize=True) for h in hops]
        pipe.run(mops, sync=True)
        barrier()
        pipe.run(mops * args.steps, sync=True)
        sm_ = pipe.stats()
        mat_ms = max_over_ranks(sm_["total_ms"]) / args.steps
        mat_exposed = sm_["exposed_compute_ms"]
        e2e_ms_total = max_over_ranks(st["total_ms"])
        e2e_step = e2e_ms_total / args.steps
        h2d_rank = sum(h.compressed_bytes for h in hops)
        d2h_rank = sum(h.rows * 4 for h in hops)
        # pinned H2D ceiling on this box (one big copy)
        big = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
        dbig = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        dbig.copy_(big, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dbig.copy_(big, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        h2d_peak = (1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9
        del big, dbig
        h2d_gbs = st["h2d_bytes"] / (st["h2d_ms"] * 1e-3) / 1e9 if st["h2d_ms"] else None
        e2e = {"value": round(world * dense_rank / (e2e_step * 1e-3) / 1e9, 2), "unit": UNIT,
               "h2d_bytes_per_step": world * h2d_rank, "d2h_bytes_per_step": world * d2h_rank,
               "ms_per_step": round(e2e_step, 4),
               "layer_ms": round(e2e_step / world, 4),
               "layers_per_step": world,
               "h2d_gbs_per_gpu": round(h2d_gbs, 2) if h2d_gbs else None,
               "h2d_pinned_peak_gbs": round(h2d_peak, 2),
               "h2d_frac_of_pcie_gen5": round(h2d_gbs / PCIE_GEN5_X16_GBS, 4) if h2d_gbs else None,
               "fused_decompress_gemv_ms_per_step": round(st["decompress_ms"] / args.steps, 4),
               "exposed_compute_ms_per_run": round(st["exposed_compute_ms"], 4),
               "materialized_w": {"layer_ms": round(mat_ms / world, 4),
                                  "value": round(world * dense_rank / (mat_ms * 1e-3) / 1e9, 2),
                                  "decompress_ms_per_step": round(sm_["decompress_ms"] / args.steps, 4),
                                  "gemv_ms_per_step": round(sm_["gemv_ms"] / args.steps, 4),
                                  "exposed_compute_ms_per_run": round(mat_exposed, 4),
                                  "note": "decompress to a dense W ring, then dense GEMV (flags bit1)"},
               "gemv_error": gemv_err,
               "api": "endor_pipeline_run (C ABI), pinned host buffers; each op y = W x by the fused "
                      "decompress -> GEMV kernel (W never in HBM)",
               "clocks": clk2.summary()}
        launches_e2e = int(st["kernel_launches"])
        # INT8 + Endor: the same layer quantized with
        # the reference's quantize_values (bit-exact on GPU), streamed as i8 values and
        # expanded by the fused dequant + decompress kernel -> f16 W -> GEMV
        if not args.no_extras:
            qops = []
            for s, h in zip(shards, hops):
                qt = E.quantize_values(s["t"])
                qops.append(HostOp(s["rows"], s["cols"], 1, h.bitmap, pinned_copy(qt.values), s["nnz"], x=h.x,
                                   y=h.y, y_host=h.y_host, quant_scale=qt.quant_scale))
            pipe.run(qops, sync=True)
            barrier()
            pipe.run(qops * args.steps, sync=True)
            sq = pipe.stats()
            q_ms = max_over_ranks(sq["total_ms"]) / args.steps
            e2e["int8_endor"] = {
                "value": round(world * dense_rank / (q_ms * 1e-3) / 1e9, 2), "unit": UNIT,
                "layer_ms": round(q_ms / world, 4), "h2d_bytes_per_step": world * sq["h2d_bytes"] // args.steps,
                "speedup_vs_f16_endor": round(e2e_step / q_ms, 3),
                "note": "values quantized to int8 (lossy, codec.hpp:306-331); f16 W rebuilt on the fly"}
        # lossless coded values (csrc/vcode.cu): low bytes raw, high bytes as k-bit dictionary codes,
        # encoded once at load time on the host; decoded on the compute stream before the fused GEMV
        if not args.no_extras:
            pipe.run(hops, sync=True)
            y_raw = [h.y_host.clone() for h in hops]
            t_enc = time.perf_counter()
            blobs = [E.encode_values(h.values) for h in hops]
            enc_s = time.perf_counter() - t_enc
            cops = [HostOp(h.rows, h.cols, 0, h.bitmap, torch.empty(0, dtype=torch.uint8), h.nnz, x=h.x, y=h.y,
                           y_host=h.y_host, vcode=bl) for h, bl in zip(hops, blobs)]
            pipe.run(cops, sync=True)
            y_same = all(torch.equal(a, h.y_host) for a, h in zip(y_raw, hops))
            barrier()
            pipe.run(cops * args.steps, sync=True)
            sc = pipe.stats()
            c_ms = max_over_ranks(sc["total_ms"]) / args.steps
            vals_raw = sum(h.values.numel() for h in hops)
            vals_coded = sum(bl.numel() for bl in blobs)
            e2e["coded_values"] = {
                "value": round(world * dense_rank / (c_ms * 1e-3) / 1e9, 2), "unit": UNIT,
                "layer_ms": round(c_ms / world, 4), "h2d_bytes_per_step": world * sc["h2d_bytes"] // args.steps,
                "speedup_vs_f16_endor": round(e2e_step / c_ms, 3),
                "values_bytes_raw": vals_raw, "values_bytes_coded": vals_coded,
                "values_ratio": round(vals_coded / vals_raw, 4),
                "modes": [E.vcode_info(bl)["mode"] for bl in blobs],
                "decode_plus_fused_gemv_ms_per_step": round(sc["decompress_ms"] / args.steps, 4),
                "exposed_compute_ms_per_run": round(sc["exposed_compute_ms"], 4),
                "host_encode_s_per_layer": round(enc_s, 3),
                "y_bit_exact_vs_raw_values": y_same,
                "note": "lossless (csrc/vcode.cu): values' high bytes as a chunked canonical Huffman stream (or "
                        "k-bit dictionary codes + exceptions, whichever is smaller), low bytes raw; the ratio depends "
                        "on the weights' exponent spread (reference synth_weight here)"}
        # the same layer with the load-time RankIndex shipped per op (prefix1024_host):
        # the fused decompress -> GEMV runs no counting / flatten pass
        if not args.no_extras:
            pre = []
            for s in shards:
                hpre = torch.empty(s["idx"].prefix.numel(), dtype=torch.int64, pin_memory=True)
                hpre.copy_(s["idx"].prefix.to(torch.int64))
                pre.append(hpre)
            iops = [HostOp(h.rows, h.cols, 0, h.bitmap, h.values, h.nnz, x=h.x, y=h.y, y_host=h.y_host,
                           prefix1024=hp) for h, hp in zip(hops, pre)]
            pipe.run(iops, sync=True)
            barrier()
            pipe.run(iops * args.steps, sync=True)
            si = pipe.stats()
            i_ms = max_over_ranks(si["total_ms"]) / args.steps
            e2e["with_index"] = {
                "layer_ms": round(i_ms / world, 4), "value": round(world * dense_rank / (i_ms * 1e-3) / 1e9, 2),
                "fused_decompress_gemv_ms_per_step": round(si["decompress_ms"] / args.steps, 4),
                "exposed_compute_ms_per_run": round(si["exposed_compute_ms"], 4),
                "h2d_bytes_per_step": world * si["h2d_bytes"] // args.steps,
                "note": "each op ships its load-time RankIndex (8 B per 1024 weights, endor_pipeline_op."
                        "prefix1024_host): 2 launches per op instead of 4"}
            # prefill: every op a GEMM over T tokens (fused tcgen05 decompress -> GEMM below the
            # two-pass threshold, decompress + dense tcgen05 GEMM above), W streamed as above
            T = int(os.environ.get("ENDOR_BENCH_PREFILL_TOKENS", "2048"))
            gx = torch.Generator(device="cpu").manual_seed(555 + rank)
            gops = []
            for s, h, hp in zip(shards, hops, pre):
                X = ((torch.rand(T, s["cols"], generator=gx) * 2 - 1).half()).to(dev)
                gops.append(HostOp(h.rows, h.cols, 0, h.bitmap, h.values, h.nnz, x=X,
                                   y=torch.empty(T, s["rows"], dtype=torch.float32, device=dev), tokens=T,
                                   prefix1024=hp))
            pipe.run(gops, sync=True)
            # parity of the last op's Y vs a float64 product over the reference-exact W
            s_last = shards[-1]
            Wl = s_last["dense"][: s_last["n"] * 2].view(torch.float16).reshape(s_last["rows"], -1)
            rs = torch.arange(0, s_last["rows"], max(1, s_last["rows"] // 64), device=dev)
            ref = gops[-1].x.double() @ Wl[rs].double().T
            mag = gops[-1].x.double().abs() @ Wl[rs].double().abs().T
            gerr = float(((gops[-1].y[:, rs].double() - ref).abs() / (mag + 1e-30)).max())
            barrier()
            reps = max(1, min(args.steps, 3))
            pipe.run(gops * reps, sync=True)
            sg = pipe.stats()
            g_ms = max_over_ranks(sg["total_ms"]) / reps
            flops = sum(2.0 * s["rows"] * s["cols"] * T for s in shards)
            gemm_ms = sg["decompress_ms"] / reps
            e2e["prefill_gemm"] = {
                "tokens": T, "layer_ms": round(g_ms / world, 4),
                "h2d_ms_per_layer": round(sg["h2d_ms"] / reps, 4),
                "gemm_ms_per_layer": round(gemm_ms, 4),
                "gemm_tflops": round(flops / (gemm_ms * 1e-3) / 1e12, 1),
                "exposed_compute_ms_per_run": round(sg["exposed_compute_ms"], 4),
                "hidden_under_h2d": bool(gemm_ms < sg["h2d_ms"] / reps),
                "max_err_over_sum_abs_sampled_rows": gerr, "within_1e-3": gerr <= 1e-3,
                "api": "endor_pipeline_run, endor_pipeline_op.tokens = T: endor_cuda_gemm_compressed per op "
                       "(tcgen05; Y stays on the device)"}
        pipe.close()

    # ---- EndorDirect: the same layer streamed from .endor files on local storage (8(f) row 2) ----
    storage = None
    if not args.no_e2e and not args.no_extras:
        import shutil
        import tempfile
        from paper_2406_11674_b200 import storage as ST
        d = tempfile.mkdtemp(prefix=f"endor_r{rank}_", dir=os.environ.get("ENDOR_BENCH_DIR", "/tmp"))
        try:
            g = torch.Generator(device="cpu").manual_seed(4321 + rank)
            fops, fbytes = [], 0
            e0 = torch.empty(0, dtype=torch.uint8)
            for i, s in enumerate(shards):
                pth = os.path.join(d, f"op{i}.endor")
                fbytes += ST.write_endor_file(s["t"], pth, version=2)  # 4 KiB-aligned sections
                x = ((torch.rand(s["cols"], generator=g) * 2 - 1).half()).to(dev)
                fops.append(HostOp(s["rows"], s["cols"], 0, e0, e0, s["nnz"], path=pth, x=x,
                                   y=torch.empty(s["rows"], dtype=torch.float32, device=dev),
                                   y_host=torch.empty(s["rows"], dtype=torch.float32, pin_memory=True)))
            sreps = max(1, min(args.steps, 2))
            fpipe = OffloadPipeline(local, nmax, ring_depth=2)
            fpipe.run(fops, sync=True)
            barrier()
            fpipe.run(fops * sreps, sync=True)
            sf = fpipe.stats()
            fpipe.close()
            r = ST.Reader(dev)
            mode = r.mode
            r.close()
            s_ms = max_over_ranks(sf["total_ms"]) / sreps
            storage = {"value": round(world * dense_rank / (s_ms * 1e-3) / 1e9, 2), "unit": UNIT,
                       "layer_ms": round(s_ms / world, 3), "layers_per_step": world, "reps": sreps,
                       "storage_gbs_per_gpu": round(sf["h2d_bytes"] / (sf["h2d_ms"] * 1e-3) / 1e9, 3),
                       "io_mode": mode, "container": "v2 (4 KiB-aligned sections, endor_file_encode_v2)",
                       "gds": "nvidia-fs not loaded on this box: O_DIRECT reads + pinned bounce buffers "
                              "(cuFile compatibility mode hangs in cuFileDriverOpen here)" if mode != "gds" else "GDS",
                       "file_bytes_per_gpu": fbytes,
                       "api": "endor_pipeline_run with endor_pipeline_op.path (C ABI)"}
            # the same layer from v3 containers (values as a lossless coded blob, decoded on the GPU)
            vops, vbytes = [], 0
            for i, (s, o) in enumerate(zip(shards, fops)):
                pth = os.path.join(d, f"op{i}_v3.endor")
                vbytes += ST.write_endor_file(s["t"], pth, version=3)
                vops.append(HostOp(o.rows, o.cols, 0, e0, e0, o.nnz, path=pth, x=o.x, y=o.y, y_host=o.y_host))
            y_v2 = [o.y_host.clone() for o in fops]
            fpipe = OffloadPipeline(local, nmax, ring_depth=2)
            fpipe.run(vops, sync=True)
            same = all(torch.equal(a, o.y_host) for a, o in zip(y_v2, vops))
            barrier()
            fpipe.run(vops * sreps, sync=True)
            sv = fpipe.stats()
            fpipe.close()
            v_ms = max_over_ranks(sv["total_ms"]) / sreps
            storage["coded_v3"] = {
                "value": round(world * dense_rank / (v_ms * 1e-3) / 1e9, 2), "unit": UNIT,
                "layer_ms": round(v_ms / world, 3), "file_bytes_per_gpu": vbytes,
                "storage_gbs_per_gpu": round(sv["h2d_bytes"] / (sv["h2d_ms"] * 1e-3) / 1e9, 3),
                "speedup_vs_v2": round(s_ms / v_ms, 3), "y_bit_exact_vs_v2": same,
                "container": "v3 (v2 layout, values section = coded-values blob, endor_file_encode_v3)"}
        finally:
            shutil.rmtree(d, ignore_errors=True)

    # ---- fused decompress -> GEMV vs decompress + GEMV, HBM-resident (8(f) row 1) -------------
    fused = None
    if not args.no_extras:
        gx = torch.Generator(device="cpu").manual_seed(77 + rank)
        xs = [((torch.rand(s["cols"], generator=gx) * 2 - 1).half()).to(dev) for s in shards]
        ys = [torch.empty(s["rows"], dtype=torch.float32, device=dev) for s in shards]

        import ctypes as C
        P, U64 = C.c_void_p, C.c_uint64
        def garr(typ, vals):
            return (typ * len(vals))(*vals)

        gem = [(garr(U64, [s["rows"] for s in g]), garr(U64, [s["cols"] for s in g]),
                garr(P, [s["out"].data.data_ptr() for s in g]),
                garr(P, [xs[gi * per_layer + j].data_ptr() for j in range(len(g))]),
                garr(P, [ys[gi * per_layer + j].data_ptr() for j in range(len(g))]), len(g))
               for gi, g in enumerate(groups)]

        def run_split():  # decompress_chunked (1 launch / layer) + batched dense GEMV (1 launch / layer)
            for p in plans_idx:
                p.launch(sp)
            for r_, c_, w_, x_, y_, n_ in gem:
                E.check(L.endor_cuda_gemv_batch(r_, c_, w_, x_, y_, None, n_, sp))

        fviews = [(_lib.TensorView * len(g))(*[s["t"].view() for s in g]) for g in groups]
        fws = torch.zeros(max(L.endor_cuda_workspace_bytes_batch(v, len(v)) for v in fviews),
                          dtype=torch.uint8, device=dev)
        fpre = [(P * len(g))(*[s["idx"].prefix.data_ptr() for s in g]) for g in groups]
        fx = [(P * len(g))(*[xs[gi * per_layer + j].data_ptr() for j in range(len(g))]) for gi, g in enumerate(groups)]
        fy = [(P * len(g))(*[ys[gi * per_layer + j].data_ptr() for j in range(len(g))]) for gi, g in enumerate(groups)]

        def run_fused():  # one endor_cuda_gemv_compressed_batch call per layer (load-time 1024 RankIndex)
            for v, pre, x, y in zip(fviews, fpre, fx, fy):
                E.check(L.endor_cuda_gemv_compressed_batch(v, pre, x, y, None, len(v), fws.data_ptr(), fws.numel(),
                                                           sp))

        def run_fused_noidx():  # no index: count + flatten + fused + row-sum launches per layer
            for v, x, y in zip(fviews, fx, fy):
                E.check(L.endor_cuda_gemv_compressed_batch(v, None, x, y, None, len(v), fws.data_ptr(), fws.numel(),
                                                           sp))

        def run_gemv_only():
            for r_, c_, w_, x_, y_, n_ in gem:
                E.check(L.endor_cuda_gemv_batch(r_, c_, w_, x_, y_, None, n_, sp))

        res = {}
        for name, fn in (("decompress_then_gemv_ms", run_split), ("fused_ms", run_fused),
                         ("fused_no_index_ms", run_fused_noidx), ("dense_gemv_ms", run_gemv_only)):
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                fn()
            b.record(stream)
            torch.cuda.synchronize()
            res[name] = max_over_ranks(a.elapsed_time(b)) / args.steps
        # HBM bytes: fused reads the compressed W (+ x, the 1024 index, y partials);
        # the dense GEMV reads the dense W
        x_bytes = sum(s["cols"] * 2 for s in shards)
        idx_bytes = sum((s["n"] // 1024) * 8 for s in shards)
        fused_bytes = comp_rank + x_bytes + idx_bytes
        fused = {"decompress_then_gemv_ms": round(res["decompress_then_gemv_ms"], 4),
                 "fused_ms": round(res["fused_ms"], 4),
                 "fused_no_index_ms": round(res["fused_no_index_ms"], 4),
                 "speedup": round(res["decompress_then_gemv_ms"] / res["fused_ms"], 3),
                 "fused_weight_gb_per_s": round(world * dense_rank / (res["fused_ms"] * 1e-3) / 1e9, 1),
                 "fused_hbm_frac": round(fused_bytes / (res["fused_ms"] * 1e-3) / 1e9 / peak, 4),
                 "dense_gemv_ms": round(res["dense_gemv_ms"], 4),
                 "dense_gemv_hbm_frac": round(dense_rank / (res["dense_gemv_ms"] * 1e-3) / 1e9 / peak, 4),
                 "note": "y = W x for the layer's six shards; fused (one batched call, load-time 1024 RankIndex) "
                         "never writes W: 1/8 + 2(1-s) B per weight read vs 5.125 for decompress + GEMV"}
        E.check(L.endor_cuda_sync_status(fws.data_ptr(), sp))
        # the fused y, element-wise against a float64 GEMV over each (bit-exact) dense shard
        run_fused()
        torch.cuda.synchronize()
        errs = [gemv_errors(y, s["out"].data.view(torch.float16).reshape(s["rows"], s["cols"]), x)
                for s, x, y in zip(shards, xs, ys)]
        fused["gemv_error"] = {"max_err_over_sum_abs": max(e["max_err_over_sum_abs"] for e in errs),
                               "max_rel_err_well_conditioned": max(e["max_rel_err_well_conditioned"] for e in errs),
                               "within_1e-3": all(e["within_1e-3"] for e in errs), "tensors": len(errs)}

    # ---- CPU baseline (rank 0, N == 1): the reference's own decompress ---------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_from_device(shards)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
                "data": "synthetic: reference synth_weight + magnitude_prune(0.5) (bit-exact on GPU), seeds 1000*layer+op",
                "config": {"workload": WORKLOAD,
                           "layers_per_step": world, "sharding": f"row-block x{world}",
                           "per_gpu_dense_bytes_per_step": dense_rank,
                           "per_gpu_compressed_bytes_per_step": comp_rank,
                           "l2": "inputs larger than L2 (no flush needed): %.2f GB/step/GPU" % ((comp_rank + dense_rank) / 1e9),
                           "parallelism": f"row-shard{world}"},
                "per_gpu_value": round(value / world, 2),
                "roofline": roofline, "decompress_no_index": no_index, "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
                "fused_decompress_gemv": fused, "storage_direct": storage,
                "gpu_launches": launches, "clocks": clk.summary() if clk else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def gemv_errors(y, W, x):
    """North star GEMV tolerance, element-wise: per row |y - y_ref| / sum_j
    |W_ij x_j| and, on rows not dominated by cancellation (|y_ref| >= 0.01 of
    that sum), |y - y_ref| / |y_ref|; y_ref in float64 on the device."""
    import torch
    Wd, xd = W.double(), x.double().to(W.device)
    ref = Wd @ xd
    mag = Wd.abs() @ xd.abs()
    err = (y.to(W.device).double() - ref).abs()
    good = (ref.abs() >= 0.01 * mag) & (mag > 0)
    out = {"max_err_over_sum_abs": float((err / mag.clamp_min(1e-30)).max()),
           "max_rel_err_well_conditioned": float((err[good] / ref[good].abs()).max()) if bool(good.any()) else 0.0,
           "rows": int(ref.numel()), "well_conditioned_rows": int(good.sum())}
    out["within_1e-3"] = out["max_err_over_sum_abs"] <= 1e-3 and out["max_rel_err_well_conditioned"] <= 1e-3
    return out


def cpu_baseline_from_device(shards):
    """Time the reference's decompress on this host: the workload's largest op
    (fc1) copied back from the device, handed to the reference."""
    import numpy as np
    from oracle import oracle as O
    R = O.ref()
    s = max(shards, key=lambda s: s["n"])
    bm = s["t"].bitmap.data.cpu().numpy().copy()
    vals = s["t"].values.cpu().numpy().copy()
    return reference_time(R, O, s["rows"], s["cols"], bm, vals, s["nnz"], reps=3,
                          sample=f"opt-66b fc1 shard {s['rows']}x{s['cols']} @50% (this run's input)")


def reference_time(R, O, rows, cols, bm, vals, nnz, reps, sample):
    import ctypes as C
    import numpy as np
    threads = os.cpu_count() or 1
    n = rows * cols
    if R is not None:
        st = C.c_int(0)
        h = R.ref_tensor_new(rows, cols, 2, bm, vals, nnz, C.byref(st))
        assert st.value == 0
        cs = 1 << 20
        chunks = (n + cs - 1) // cs
        pref = np.zeros(chunks, np.uint64)
        R.ref_rank_index(bm, n, cs, pref)
        dst = np.ones(n * 2, np.uint8)  # pre-faulted
        times = []
        for _ in range(reps):
            t = R.ref_decompress_parallel_timed(h, pref, cs, chunks, threads, dst.ctypes.data, C.byref(st))
            times.append(t)
        t1 = R.ref_decompress_timed(h, None, C.byref(st))
        R.ref_tensor_free(h)
        kind = "reference"
    else:
        cs = 1 << 20
        _, pref = O.rank_index(bm, n, cs)
        dst = np.ones(n * 2, np.uint8)
        times = [O.lib().or_decompress_parallel(n, 2, bm, vals, cs, pref, dst, threads) for _ in range(reps)]
        t1 = None
        kind = "port"
    best = min(times)
    return {"value": round(n * 2 / best / 1e9, 3), "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{sample}: decompress_chunk_into fan-out over {threads} threads, chunk 2^20, best of {reps}",
            "single_thread_decompress_gbs": round(n * 2 / t1 / 1e9, 3) if t1 else None}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    import ctypes as C
    import numpy as np
    world, rank, _ = env_dist()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2406_11674_b200 import catalog
    R = O.ref()
    L = O.lib()
    L.or_make_op_mt.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_int, O._u8p, O._u8p]
    L.or_make_op_mt.restype = C.c_uint64
    threads = os.cpu_count() or 1
    spec = catalog.model_catalog("opt-66b")
    ops = []
    for oi, op in enumerate(spec.ops):  # one full layer (layer 0), generated on the CPU
        n = op.rows * op.cols
        bm = np.zeros((n + 7) // 8, np.uint8)
        vals = np.zeros(n * 2, np.uint8)
        nnz = L.or_make_op_mt(op.rows, op.cols, catalog.op_seed(0, oi), SPARSITY, threads, bm, vals)
        vals = vals[: nnz * 2].copy()
        st = C.c_int(0)
        h = R.ref_tensor_new(op.rows, op.cols, 2, bm, vals, nnz, C.byref(st)) if R else None
        cs = 1 << 20
        chunks = (n + cs - 1) // cs
        pref = np.zeros(chunks, np.uint64)
        if R:
            R.ref_rank_index(bm, n, cs, pref)
        else:
            _, pref = O.rank_index(bm, n, cs)
        ops.append(dict(n=n, bm=bm, vals=vals, nnz=nnz, h=h, pref=pref, chunks=chunks,
                        dst=np.ones(n * 2, np.uint8)))

    def step():
        t = 0.0
        st = C.c_int(0)
        for o in ops:
            if R:
                t += R.ref_decompress_parallel_timed(o["h"], o["pref"], 1 << 20, o["chunks"], threads,
                                                     o["dst"].ctypes.data, C.byref(st))
            else:
                t += L.or_decompress_parallel(o["n"], 2, o["bm"], o["vals"], 1 << 20, o["pref"], o["dst"],
                                              threads)
        return t

    for _ in range(args.warmup):
        step()
    total = sum(step() for _ in range(args.steps))
    dense = sum(o["n"] * 2 for o in ops)
    ms = total / args.steps * 1e3
    value = dense / (ms * 1e-3) / 1e9
    kind = "reference" if R else "port"
    sample = (f"one full opt-66b layer (6 ops, {dense / 1e9:.2f} GB dense) per step; "
              f"decompress_chunk_into (codec.hpp:191) over {threads} threads, chunk 2^20")
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic (reference synth_weight + magnitude_prune 0.5)",
            "config": {"workload": WORKLOAD, "layers_per_step": 1,
                       "parallelism": f"{threads} host threads"},
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    for o in ops:
        if o["h"]:
            R.ref_tensor_free(o["h"])
    print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n: int, argv) -> int:
    """Re-run this script as N ranks under torch.distributed.run (the same
    launch the driver uses for N>1) and return the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the INT8 pipeline and fused-GEMV side measurements")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `bench.py --gpus N` outside a launcher: become the launcher -- one
        # process per GPU under torchrun (NCCL rendezvous on 127.0.0.1); rank 0
        # prints the single JSON line
        sys.exit(relaunch(args.gpus, sys.argv[1:]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
