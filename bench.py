#!/usr/bin/env python
"""bench.py -- spGEMM GFLOPS (2 x intermediate products / device time).

Workload (default): C = A.A, A = R-MAT power-law graph, 2^20 rows, edge
factor 16, (a,b,c,d) = (0.45,0.15,0.15,0.25) -- BASELINE.json configs[2],
the largest single-GPU configuration (575M filtered tile pairs, 583M output
nonzeros; BASELINE's metric names no config, so the largest one that fits a
GPU is the headline).  fp16 in / fp32 accumulate, synthetic (generated
deterministically, no dataset).  The other configs (--config
poisson|fem27|rect|amg) are parity cases and extra lines.

A "step" is one full spGEMM: CSR A (and B) resident in HBM -> CSR C in HBM,
through the C ABI (tsg_spgemm), with every phase, allocation and size
readback inside the timed region (PAPER.md:585 counts allocations).  L2
(126 MB) is flushed with a 256 MB write before every timed step, outside the
timed span.  `e2e` is the same call with pinned HOST CSR in and host CSR out
(H2D + D2H inside the timed region).

  python bench.py [--gpus N --steps K --warmup W] [--config rmat]
  python bench.py --impl reference ...   (the reference CPU implementation)

N > 1 (torchrun, one rank per GPU, NCCL): A is split into tile-row panels
balanced by work (intermediate products per tile row); B is broadcast from
rank 0 over NVLink each step (the exchange step of SURVEY.md 8(e)); value =
total flops of all ranks / max over ranks of the step time.  Total work is
fixed: "scaling": "strong".

The CPU legs (cpu_baseline, --impl reference) time the reference compiled in
place (oracle/_ref) on the host cores.  R-MAT takes minutes per full CPU run,
so they time a bounded sample: every 64th tile row of A times the full B
(~6.5% of the products, ~15-25 s per run); GFLOPS are the sample's own flops
over its time.
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

from pathlib import Path

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "spGEMM GFLOPS (2x intermediate products / device time)"
CONFIG_TEXT = {
    "poisson": "C = A.A, 2D 5-point Poisson 256x256 (65,536 rows)",
    "fem27": "C = A.A, 3D 27-point FEM-like stencil 64^3 (262,144 rows, 6.86M nnz)",
    "rmat": "C = A.A, R-MAT 2^20 rows, edge factor 16, (0.45,0.15,0.15,0.25)",
    "rect": "C = A.B, 1M x 500k . 500k x 1M, density 1e-5",
    "amg": "C = (R.A).P, 7-point Laplacian 128^3, trilinear prolongation",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="rmat", choices=list(CONFIG_TEXT))
    p.add_argument("--mode", default="tensor", choices=["tensor", "ordered"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-runs", type=int, default=3)
    p.add_argument("--no-e2e", action="store_true", help="skip the host-to-host e2e measurement")
    p.add_argument("--no-cpu-extra", action="store_true",
                   help="skip the threads=1 / pairing-off / Gustavson CPU points")
    return p.parse_args()


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
class Clocks:
    """SM clock and clock-event reasons sampled every ~2 ms during the timed
    region through NVML (nvidia-smi's ~100 ms per query is too coarse for a
    region of a few tens of ms); falls back to nvidia-smi."""

    REASONS = {  # NVML clocks-event-reason bits
        "hw_slowdown": 0x0000000000000008, "sw_thermal_slowdown": 0x0000000000000020,
        "hw_thermal_slowdown": 0x0000000000000040, "sw_power_cap": 0x0000000000000004,
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, rs))
                self._stop.wait(0.002)
            self._nvml = True
        except Exception:
            self._nvml = False
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    sm, mx, rs = [x.strip() for x in out.split(",")]
                    self.samples.append((float(sm), float(mx), int(rs, 16)))
                except Exception:
                    pass
                self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        sm = [x[0] for x in self.samples]
        reasons = sorted({n for x in self.samples for n, b in self.REASONS.items() if x[2] & b})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------
def operands(config):
    from paper_2009_14600_b200 import workloads as W
    return W.make(config)


def algorithmic_bytes(st, nnzA, nnzB, rowsA, rowsC, same):
    """SURVEY.md 8(d) compulsory-traffic model per phase (T=16 tiles:
    tile record 32 B mask + 8 B coords + 4 B offset, fp16 in, fp32 out, 8 B pairs)."""
    tA, tB = st["tiles_a"], st["tiles_b"]
    P, S, cnt, nnzC = st["filtered_pairs"], st["segments"], st["counted_elements"], st["nnz_c"]
    conv = (8 * (rowsA + 1) + 8 * nnzA) + (44 * tA + 2 * nnzA)
    if not same:
        conv += (8 * (rowsA + 1) + 8 * nnzB) + (44 * tB + 2 * nnzB)
    return {
        "convert": conv,
        "task_list": 40 * (tA + tB) + 8 * P,      # enumerate + filter (tile metadata in, pairs out)
        "sort": 16 * P + 8 * S,                    # read + write pairs, segment table
        "counting": 0,                             # fused into the numeric kernel (no own traffic)
        # SURVEY numeric bytes (the fused kernel also does the counting pass on
        # the same operands, so the operand bytes are not counted twice)
        "multiply": 8 * P + 44 * (tA + tB) + 2 * (nnzA + nnzB) + 44 * S + 4 * cnt,
        # SURVEY output bytes: tiled C in, CSR out (tC ~ S output tiles)
        "compaction": 44 * S + 4 * nnzC + 8 * (rowsC + 1) + 8 * nnzC,
    }


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2009_14600_b200 import _lib as L
    from paper_2009_14600_b200 import workloads as W
    from paper_2009_14600_b200.tilemul import Context, Csr, _view

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; TSG_DIST_BACKEND=gloo (with ranks sharing GPUs modulo
    # the device count) exists only to exercise this path on a 1-GPU box
    backend = os.environ.get("TSG_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    # a dedicated stream shared by the library and the timing events: every
    # kernel of the step is launched on the stream the events are recorded on
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = Context(device=local, stream=stream.cuda_stream)

    mats = operands(args.config)
    chain = len(mats) == 3
    if chain:
        Afull, Bs = mats[0], mats[1:]
    elif len(mats) == 2:
        Afull, Bs = mats[0], [mats[1]]
    else:
        Afull, Bs = mats[0], [mats[0]]
    same = len(mats) == 1 and world == 1

    # rank panel of A: tile-row aligned row ranges balanced by work
    # (paper_2009_14600_b200/distributed.py)
    from paper_2009_14600_b200 import distributed as D
    r0, r1 = D.panel_bounds(Afull, Bs[0], world)[rank]
    Apanel = D.take_rows(Afull, r0, r1)

    # flops of this rank: 2 * C-bar over the chain stages (computed, never hard-coded)
    cb = W.cbar(Apanel, Bs[0])
    if chain:  # second stage C-bar needs the structure of R.A (untimed setup)
        RA = ctx.spgemm(Apanel, Bs[0]).C
        cb += W.cbar(RA, Bs[1])
    keep = []

    import torch

    def dev_csr(M):
        """Device CSR in one flat buffer (row_ptr | col | val, so a broadcast
        is one collective); the workloads' binary16 values travel as fp16
        when that is exact (TSG_DEV_F16=0: fp32)."""
        val = torch.from_numpy(np.ascontiguousarray(M.val))
        if os.environ.get("TSG_DEV_F16", "1") == "1":
            h = val.to(torch.float16)
            if torch.equal(h.to(val.dtype), val):
                val = h
        parts = [torch.from_numpy(np.ascontiguousarray(M.row_ptr, dtype=np.int64)),
                 torch.from_numpy(np.ascontiguousarray(M.col, dtype=np.int32)), val]
        sizes = [t.numel() * t.element_size() for t in parts]
        pads = [(n + 7) // 8 * 8 for n in sizes]  # every part 8-byte aligned (f64 values)
        flat = torch.empty(sum(pads), dtype=torch.uint8, device=dev)
        views, o = [], 0
        for t, n, pn in zip(parts, sizes, pads):
            v = flat[o:o + n].view(t.dtype)
            v.copy_(t.to(dev))
            views.append(v)
            o += pn
        return Csr(M.rows, M.cols, *views), flat

    A_dev, _ = dev_csr(Apanel)
    a_view = _view(A_dev, keep)
    # B lives on rank 0 and is broadcast each step (N>1, one collective per
    # operand); same-pointer view for A.A at N=1
    B_pack = [dev_csr(B) for B in Bs]
    B_dev = [b for b, _ in B_pack]
    b_views = [a_view] if same else [_view(B, keep) for B in B_dev]
    opts = L.tsg_options()
    ctx._lib.tsg_default_options(opts)
    opts.mode = L.TSG_MODE_ORDERED if args.mode == "ordered" else L.TSG_MODE_TENSOR

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # general-row configs at N > 1: B's tile summary is split over the ranks
    # (each summarises its row panel of B) and all-gathered, instead of every
    # rank converting all of B (distributed.gather_b_summary; TSG_BSUM=0: off)
    use_bsum = world > 1 and not chain and args.config in ("rmat", "rect") and \
        os.environ.get("TSG_BSUM", "1") == "1"
    if use_bsum:
        bb0, bb1 = D.b_panel_bounds(Bs[0], world)[rank]
        brp = np.asarray(Bs[0].row_ptr)
        blo, bhi = int(brp[bb0]), int(brp[bb1])

    def b_summary():
        Bd = B_dev[0]
        Bp = Csr(bb1 - bb0, Bd.cols, Bd.row_ptr[bb0:bb1 + 1] - blo, Bd.col[blo:bhi], Bd.val[blo:bhi])
        part = ctx.b_summary(Bp)
        full = D.gather_b_summary(part, dist, dev)
        return part, full

    def one_step(stats=None):
        if world > 1:
            for _, flat in B_pack:
                dist.broadcast(flat, src=0)
        if use_bsum:
            part, full = b_summary()
            co = L.tsg_csr_out()
            co.mem = L.TSG_MEM_DEVICE
            rc = ctx.spgemm_bsum_raw(a_view, b_views[0], full, opts, co, stats)
            part.free()
            if rc != 0:
                raise RuntimeError(ctx._lib.tsg_last_error(ctx.handle).decode())
            return co
        if chain:
            import ctypes as C
            arr = (C.POINTER(L.tsg_csr) * 3)(C.pointer(a_view), C.pointer(b_views[0]), C.pointer(b_views[1]))
            co = L.tsg_csr_out()
            co.mem = L.TSG_MEM_DEVICE
            rc = ctx._lib.tsg_spgemm_chain(ctx.handle, 3, arr, C.byref(co), C.byref(opts),
                                           C.byref(stats) if stats is not None else None)
        else:
            co = L.tsg_csr_out()
            co.mem = L.TSG_MEM_DEVICE
            rc = ctx.spgemm_raw(a_view, b_views[0], opts, co, stats)
        if rc != 0:
            raise RuntimeError(ctx._lib.tsg_last_error(ctx.handle).decode())
        return co

    def timed(k, fn):
        times = []
        for _ in range(k):
            flush.fill_(1.0)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            if out is not None:
                ctx.free(out)
        return times

    for _ in range(args.warmup):
        ctx.free(one_step())
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    with Clocks(local) as clk:
        times = timed(args.steps, one_step)
    launches = ctx.launch_count() - launches0
    ms = float(np.mean(times))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
        c = torch.tensor([cb], dtype=torch.float64, device=dev)
        dist.all_reduce(c)
        cb_total = int(c.item())
    else:
        ms_max, cb_total = ms, cb
    value = 2.0 * cb_total / (ms_max * 1e-3) / 1e9

    # ---- per-phase device times (separate run, phase events on) -> roofline
    st = L.tsg_run_stats()
    opts.phase_timing = 1
    phase_ms = {}
    for _ in range(3):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        st = L.tsg_run_stats()
        ctx.free(one_step(st))
        for ph in ("convert", "task_list", "sort", "counting", "multiply", "compaction", "total"):
            phase_ms.setdefault(ph, []).append(ctx.last_phase_ms(ph) if not chain else getattr(st, ph) * 1e3)
        phase_ms.setdefault("numeric_kernel", []).append(ctx.last_phase_ms("numeric_kernel"))
        phase_ms.setdefault("assemble_kernel", []).append(ctx.last_phase_ms("assemble_kernel"))
    opts.phase_timing = 0
    phase_ms = {k: float(np.median(v)) for k, v in phase_ms.items()}
    sd = st.as_dict()
    nnzB = Bs[0].nnz
    bytes_ = algorithmic_bytes(sd, Apanel.nnz, nnzB, Apanel.rows, Apanel.rows, same)
    peaks = json.loads((Path(ROOT) / "MEASURED_PEAKS.json").read_text()) if (Path(ROOT) / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # dominant kernel: the fused numeric pass -- light rows: panel_numeric_kernel
    # (task list + counting + SEaC multiply of each tile row, tsg_panel.cu);
    # general rows: esc_kernel (enumerate + sort + count + multiply of each
    # work unit in shared memory, tsg_esc.cu).  Its time is the CUDA-event
    # bracket of that one kernel launch on the library's stream (kev[0..1]).
    # achieved = SURVEY 8(d) "numeric" bytes / that time (conservative: the
    # fused kernel also performs the task-list and sort phases, whose SURVEY
    # bytes are reported separately as achieved_fused_phases).
    dom = "multiply"
    kms = phase_ms.get("numeric_kernel") or phase_ms.get(dom)
    achieved = bytes_[dom] / (kms * 1e-3) / 1e9 if kms else 0.0
    fused_bytes = bytes_["task_list"] + bytes_["sort"] + bytes_["multiply"]
    achieved_fused = fused_bytes / (kms * 1e-3) / 1e9 if kms else 0.0
    kname = L.PATH_KERNEL[sd["path"]]
    traffic, prof_name = None, None
    for rnd in ("r02", "r01"):
        cand = Path(ROOT) / f"profiles/{rnd}_ncu_full_{args.config}.json"
        if cand.exists():
            prof_name = str(cand.relative_to(ROOT))
            break
    if world == 1 and prof_name:
        kk = json.loads((Path(ROOT) / prof_name).read_text())["kernels"]
        tot = [k["dram_read_bytes"] + k["dram_write_bytes"] for name, k in kk.items()
               if name.split("<")[0].split("#")[0].split("::")[-1] == kname]
        traffic = int(sum(tot) / len(tot)) if tot else None

    # ---- e2e: host CSR in (pinned), host CSR out, through the public API
    pin = []
    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        pin.append(t)
        return t
    def host_vals(v):
        # the workloads are binary16-valued (fp16 in): ship binary16 bits over
        # PCIe when that is exact (tsg_csr dtype TSG_F16), else fp32
        v = np.asarray(v)
        h = v.astype(np.float16)
        return pinned(h.view(np.int16)).numpy().view(np.float16) if np.array_equal(h.astype(v.dtype), v) else pinned(v).numpy()
    Ah = Csr(Apanel.rows, Apanel.cols, pinned(Apanel.row_ptr).numpy(), pinned(Apanel.col).numpy(),
             host_vals(Apanel.val))
    Bh = [Csr(B.rows, B.cols, pinned(B.row_ptr).numpy(), pinned(B.col).numpy(), host_vals(B.val)) for B in Bs]
    e2e_stats = {}

    def e2e_step():
        import ctypes as C
        keep2 = []
        av = _view(Ah, keep2)
        bvs = [av] if same else [_view(B, keep2) for B in Bh]
        co = L.tsg_csr_out()
        co.mem = L.TSG_MEM_HOST
        st2 = L.tsg_run_stats()
        if chain:
            arr = (C.POINTER(L.tsg_csr) * 3)(C.pointer(av), C.pointer(bvs[0]), C.pointer(bvs[1]))
            rc = ctx._lib.tsg_spgemm_chain(ctx.handle, 3, arr, C.byref(co), C.byref(opts), C.byref(st2))
        else:
            rc = ctx.spgemm_raw(av, bvs[0], opts, co, st2)
        if rc != 0:
            raise RuntimeError(ctx._lib.tsg_last_error(ctx.handle).decode())
        e2e_stats["h2d"] = int(st2.h2d_bytes)
        e2e_stats["d2h"] = int(st2.d2h_bytes)
        return co

    if args.no_e2e:
        e2e_times = [float("nan")]
    else:
        for _ in range(2):
            ctx.free(e2e_step())
        e2e_times = timed(max(3, args.steps // 2), e2e_step)
    e2e_ms = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = 2.0 * cb_total / (e2e_ms * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f16-in/f32-acc",
        "data": "synthetic (deterministic generator, paper_2009_14600_b200/workloads.py)",
        "config": config_key(args.config, cb_total, Afull.nnz),
        "details": {"mode": args.mode,
                    "parallelism": (f"A tile-row panels x{world}, B broadcast"
                                    + (" + B-summary all-gather" if use_bsum else "")) if world > 1 else "single GPU",
                    "l2": "flushed (256 MB write) before every timed step",
                    "values_at_boundary": "binary16 bits (TSG_F16) when exact, on the device and over PCIe",
                    "nnz_c": sd["nnz_c"], "tiles_a": sd["tiles_a"], "raw_pairs": sd["raw_pairs"],
                    "filtered_pairs": sd["filtered_pairs"], "segments": sd["segments"],
                    "counted_elements": sd["counted_elements"], "path": kname,
                    "device_mem_peak_bytes": sd["mem_peak"]},
        "e2e": {"value": round(e2e_value, 3), "unit": "GFLOPS", "ms_per_step": round(e2e_ms, 4),
                "h2d_bytes_per_step": e2e_stats.get("h2d"), "d2h_bytes_per_step": e2e_stats.get("d2h")},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / max(1, args.steps),
        "phase_ms": {k: round(v, 4) for k, v in phase_ms.items()},
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1),
                     "achieved_fused_phases": round(achieved_fused, 1), "fused_phase_bytes": int(fused_bytes),
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "kernel_ms": round(kms, 4) if kms else None, "algorithmic_bytes": int(bytes_[dom]),
                     "traffic": traffic, "traffic_source": f"{prof_name} (ncu --set full)" if traffic else None},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, mats, 2 * cb_total)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


# Bounded CPU samples: every `stride`-th tile row of the first operand
# (workloads.sample_tile_rows) times the full other operands.  R-MAT takes
# minutes per full reference run (133.6 s on 8 threads), the
# others finish in seconds and run whole.
CPU_SAMPLE_STRIDE = {"rmat": 64}


def cpu_sample(config, mats):
    from paper_2009_14600_b200 import workloads as W
    stride = CPU_SAMPLE_STRIDE.get(config, 1)
    if stride == 1:
        return mats, "the whole workload"
    S = W.sample_tile_rows(mats[0], stride)
    return ([S] + list(mats[1:]) if len(mats) > 1 else [S, mats[0]]), \
        f"every {stride}th 16-row tile row of A ({S.rows} rows, {S.nnz} nnz) times the full B"


def cpu_run(mats, threads):
    """The reference: spgemm_square(A) for one operand, the pass composition
    (kernels.cpp:222-302 phases) for A.B, the chain with the binary16
    downcast for three."""
    from oracle import ref
    if len(mats) == 1:
        return ref.spgemm(mats[0], threads=threads)
    if len(mats) == 2:
        return ref.spgemm(mats[0], mats[1], threads=threads)
    return ref.chain(mats, threads=threads)


def sample_flops(smats):
    from paper_2009_14600_b200 import workloads as W
    from paper_2009_14600_b200.tilemul import Csr
    if len(smats) == 1:
        return 2 * W.cbar(smats[0], smats[0])
    cb = W.cbar(smats[0], smats[1])
    if len(smats) == 3:
        RA = cpu_run(smats[:2], 1)  # only to size the second stage's C-bar (untimed)
        cb += W.cbar(Csr(RA.rows, RA.cols, RA.row_ptr, RA.col, RA.val), smats[2])
    return 2 * cb


def cpu_baseline(args, mats, flops):
    """The reference tilemul (oracle/_ref, compiled unmodified) on host cores,
    on a bounded sample of the workload."""
    from oracle import ref
    if not ref.available():
        return {"value": None, "unavailable": "oracle/_ref/libref_tilemul.so not built"}
    cores = os.cpu_count() or 1
    smats, what = cpu_sample(args.config, mats)
    sflops = flops if smats is mats else sample_flops(smats)
    runs = 1 if smats is not mats else max(1, args.cpu_sample_runs)
    secs = [cpu_run(smats, threads=cores).times["total"] for _ in range(runs)]
    s = statistics.median(secs)
    out = {"value": round(sflops / s / 1e9, 4), "unit": "GFLOPS", "cores": cores, "kind": "reference",
           "cpu_model": cpu_model(),
           "sample": f"{what}: {sflops} flops; {len(secs)} run(s) of the reference "
                     f"(spgemm_square / pass composition, pairing on, threads={cores}), median {s:.3f} s; "
                     f"input tiling untimed (SPEC.md:522)"}
    # one thread, pairing off, and the single-threaded
    # Gustavson mixed oracle (dense_spgemm_mixed_ordered), one run each on the
    # same sample
    if not args.no_cpu_extra and len(smats) <= 2:
        def gf(t):
            return round(sflops / t / 1e9, 4)
        t1 = cpu_run(smats, threads=1).times["total"]
        tp = (ref.spgemm(smats[0], threads=cores, pairing=False) if len(smats) == 1 else
              ref.spgemm(smats[0], smats[1], threads=cores, pairing=False)).times["total"]
        to = ref.oracle(smats[0], smats[1] if len(smats) > 1 else None).times["total"]
        out["extra_points"] = {"threads_1": gf(t1), f"pairing_off_threads_{cores}": gf(tp),
                               "gustavson_mixed_oracle_threads_1": gf(to), "unit": "GFLOPS"}
    return out


def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def config_key(config, cb_total, nnz_a):
    """The workload identity both arms print (same keys and values)."""
    return {"workload": CONFIG_TEXT[config], "config": config, "flops_per_step": 2 * cb_total,
            "cbar": cb_total, "nnz_a": nnz_a}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref_tilemul.so not built"}))
        return
    from paper_2009_14600_b200 import workloads as W
    from paper_2009_14600_b200.tilemul import Csr
    mats = operands(args.config)
    cb = W.cbar(mats[0], mats[1] if len(mats) > 1 else mats[0])
    if len(mats) == 3:
        RA = cpu_run(mats[:2], 1)  # only to size the second stage's C-bar
        cb += W.cbar(Csr(RA.rows, RA.cols, RA.row_ptr, RA.col, RA.val), mats[2])
    smats, what = cpu_sample(args.config, mats)
    sflops = 2 * cb if smats is mats else sample_flops(smats)
    cores = os.cpu_count() or 1
    # bounded: a FEM27 run is ~1.8 s on 16 host threads, an R-MAT sample ~15-25 s;
    # K <= 10 (<= 3 for a sampled workload), W <= 3 (<= 1) keep the arm to minutes
    cap_k, cap_w = (10, 3) if smats is mats else (3, 1)
    steps = max(1, min(args.steps, cap_k))
    warm = max(0, min(args.warmup, cap_w))
    for _ in range(warm):
        cpu_run(smats, cores)
    secs = [cpu_run(smats, cores).times["total"] for _ in range(steps)]
    s = float(np.mean(secs))
    v = sflops / s / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GFLOPS", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": round(s * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16-in/f32-acc (CPU, sequential fp32)",
        "data": "synthetic", "config": config_key(args.config, cb, mats[0].nnz),
        "cpu_baseline": {"value": round(v, 4), "unit": "GFLOPS", "cores": cores, "kind": "reference",
                         "sample": f"{what}: {sflops} flops per step; {steps} step(s) after {warm} warm-up "
                                   f"(steps capped at {cap_k}, warm-up at {cap_w}); pairing on, threads={cores}"},
        "e2e": {"value": round(v, 4), "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
