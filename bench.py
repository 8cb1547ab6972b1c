"""Benchmark of the B200 Flash All-Reduce (BASELINE.json metric:
"all-reduce latency & effective GB/s at TP=2/4/8 vs NCCL bf16; roofline
fraction").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1|c4]

N=1 (the driver default): the headline workload C2 — INT4 asym g128 flash
all-reduce of bf16 [8,1024,8192] per rank at TP=8 — with all 8 TP ranks
emulated on one B200 (8 logical ranks, the reference's list-of-tensors call;
peer stores land in local HBM instead of crossing NVLink). One step = one
all-reduce of all 8 ranks' tensors = one launch of the fused persistent
kernel. N>1 (torchrun): one rank per GPU over CUDA IPC / NVLink with
NCCL bf16 all_reduce timed beside it.

value = sum over TP ranks of the bf16 input bytes all-reduced per second
(whole job); algbw (nccl-tests convention, e*M/t) and latency are reported
too. Inputs (1 GiB at N=1) exceed the 126 MB L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (tp, tokens-per-rank shape, bits, dtype)
    "c2": dict(tp=8, shape=(8, 1024, 8192), bits=4, group=128, dtype="bf16",
               desc="INT4 asym g128 flash all-reduce of bf16 [8,1024,8192] per rank at TP=8 (Llama-3-70B prefill)"),
    "c1": dict(tp=4, shape=(1024, 8192), bits=8, group=128, dtype="fp16",
               desc="INT8 asym g128 flash all-reduce of fp16 [1024,8192] per rank at TP=4"),
    "c4": dict(tp=8, shape=(64, 8192), bits=4, group=128, dtype="bf16",
               desc="decode: INT4 g128 flash all-reduce of bf16 [64,8192] per rank at TP=8 (latency-bound)"),
}


def load_peaks() -> dict:
    """HBM copy peak: MEASURED_PEAKS.json (driver-written on this pool) if present,
    else the fallback of B200_PROFILING.md (6.65 TB/s)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            with open(p) as fh:
                d = json.load(fh)
            flat = {}

            def walk(o, pre=""):
                if isinstance(o, dict):
                    for k, v in o.items():
                        walk(v, pre + k + ".")
                elif isinstance(o, (int, float)):
                    flat[pre[:-1]] = float(o)

            walk(d)
            for k in ("hbm_gbs", "hbm.gbs", "hbm_GBps"):
                if k in flat:
                    return {"hbm_gbs": flat[k], "source": f"measured (MEASURED_PEAKS.json {k})"}
            for k, v in flat.items():
                if "hbm" in k.lower() and "gb" in k.lower() and v > 100:
                    return {"hbm_gbs": v, "source": f"measured (MEASURED_PEAKS.json {k})"}
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


class NvmlClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~1 ms from a background thread DURING the timed region (a 20-step C2 run is
    ~12 ms, shorter than nvidia-smi's sampling period). Falls back to the
    nvidia-smi sampler when NVML is unavailable."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop_flag = threading.Event()
        self.thread = None
        self.fallback = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            masks = [(nm, getattr(pynvml, attr, 0)) for nm, attr in self.NAMES]

            def run():
                while not self.stop_flag.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                        rs = get_reasons(self.h)
                        self.samples.append((sm, [nm for nm, m in masks if m and (rs & m)]))
                    except Exception:
                        pass
                    time.sleep(0.001)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self.fallback = ClockSampler(self.index)
            self.fallback.start()

    def stop(self) -> dict:
        if self.fallback is not None:
            return self.fallback.stop()
        self.stop_flag.set()
        self.thread.join(timeout=2)
        sms = [sm for sm, _ in self.samples]
        reasons = sorted({r for _, rs in self.samples for r in rs})
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(sms), "source": "nvml, ~1 ms period"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sms.append(float(parts[1]))
                    maxes.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def wire_len(bits: int, group: int, n: int) -> int:
    packed = (n * (4 if bits <= 4 else 8) + 7) // 8
    return packed + (-(-n // group)) * 3


# ---------------------------------------------------------------------------
# CPU baseline: the reference's algorithm (oracle port, test infrastructure) on
# the host cores. Owners' segments are independent (collectives.py:355-386) and
# results are chunk-transparent at group multiples (collectives.py:14-16), so
# the sample is split into (owner, piece) jobs run by a fork pool on every core.

_REF = {}


def _ref_job(job):
    from oracle import flash_oracle as orc

    j, lo, hi = job
    xs, c1, c2, seg = _REF["xs"], _REF["c1"], _REF["c2"], _REF["seg"]
    parts = [orc.dequantize(orc.quantize(x[j * seg + lo: j * seg + hi], c1)) for x in xs]
    red = orc.sequential_sum(parts)  # ascending source rank (collectives.py:182-187)
    return orc.dequantize(orc.quantize(red, c2))


def cpu_reference_run(tp: int, elems: int, bits: int, group: int, workers: int, seed: int = 0):
    """One flash all-reduce of `tp` ranks x `elems` elements through the oracle
    port, split over `workers` processes. Returns (seconds, output of rank 0)."""
    import multiprocessing as mp

    import numpy as np

    from oracle import flash_oracle as orc

    rng = np.random.default_rng(seed)
    seg = -(-elems // tp)
    xs = [np.pad(rng.standard_normal(elems).astype(np.float32), (0, tp * seg - elems)) for _ in range(tp)]
    c = orc.Codec(bits=bits, group_size=group)
    _REF.update(xs=xs, c1=c, c2=c, seg=seg)
    pieces = max(1, -(-workers // tp))
    per = -(-(-(-seg // pieces)) // group) * group
    jobs = [(j, lo, min(seg, lo + per)) for j in range(tp) for lo in range(0, seg, per)]
    t0 = time.perf_counter()
    if workers <= 1:
        outs = [_ref_job(jb) for jb in jobs]
    else:
        with mp.get_context("fork").Pool(workers) as pool:
            outs = pool.map(_ref_job, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    return dt, np.concatenate(outs)[:elems]


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_sample_elems(cfg: dict) -> int:
    # bounded sample: 1/16 of the C2 per-rank tensor (4,194,304 elements per rank)
    m = math.prod(cfg["shape"])
    return max(cfg["tp"] * 1024, min(m, 1 << 22))


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    elems = cpu_sample_elems(cfg)
    e = 2
    workers = host_threads()
    times = []
    for i in range(args.warmup + args.steps):
        dt, _ = cpu_reference_run(cfg["tp"], elems, cfg["bits"], cfg["group"], workers, seed=i)
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    val = cfg["tp"] * e * elems / t / 1e9
    sample = (f"{cfg['tp']} ranks x {elems} elements per rank ({elems / math.prod(cfg['shape']):.4f} of the "
              f"per-rank tensor), fp32 arrays of bf16-valued work")
    note = (f"oracle/flash_oracle.py numpy restatement of qcollectives.flash_all_reduce (the reference is Python "
            f"and cannot travel to the GPU box), (owner, piece) jobs on a {workers}-process fork pool")
    line = {"impl": "reference", "metric": args.metric, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "tp": cfg["tp"], "sample": sample},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": workers, "kind": "port", "sample": sample,
                             "host_cpus": os.cpu_count(), "note": note},
            "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


def _dtype(name):
    import torch

    return {"bf16": torch.bfloat16, "fp16": torch.float16}[name]


def _wall_time(fn, steps) -> float:
    """ms per call of a BLOCKING call (it synchronises its own streams), host clock."""
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e3


def _events_time(fn, steps, stream):
    """(average ms, list of per-step ms) of `steps` calls, CUDA events on `stream`."""
    import torch

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    torch.cuda.synchronize()
    evs[0].record(stream)
    for i in range(steps):
        fn()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    return evs[0].elapsed_time(evs[-1]) / steps, per


def graph_time(fn, reps, stream) -> float:
    """Average device ms of one `fn` call: `reps` calls captured in a CUDA graph,
    the graph replayed 5 times between CUDA events."""
    import torch

    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(5):
        gr.replay()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (5 * reps)


def load_traffic() -> dict:
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


def bench_local(args, cfg, peaks):
    """N=1: all TP ranks as logical ranks of one B200."""
    import torch

    import paper_2412_04964_b200 as fc
    from paper_2412_04964_b200 import _lib
    from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    tp, dt = cfg["tp"], _dtype(cfg["dtype"])
    m = math.prod(cfg["shape"])
    e = 2
    seg = -(-m // tp)
    fcfg = fc.FlashConfig.from_bits(cfg["bits"], group_size=cfg["group"])
    comm = FlashComm.local([0] * tp, slot_bytes_for(seg, fcfg.stage1_codec, fcfg.stage2_codec))
    if args.ctas:
        comm.set_option(_lib.OPT_CTAS, args.ctas)
    if args.lag:
        comm.set_option(_lib.OPT_LAG, args.lag)
    if args.fused:
        comm.set_option(_lib.OPT_FUSED, 1)
    g = torch.Generator(device=dev).manual_seed(1234)
    ins = [torch.randn(m, device=dev, generator=g).to(dt) for _ in range(tp)]
    outs = [torch.empty(m, device=dev, dtype=dt) for _ in range(tp)]
    stream = torch.cuda.current_stream(dev)
    step = lambda: comm.all_reduce_local(ins, fcfg, outs=outs, check=False)  # noqa: E731
    for _ in range(args.warmup):
        step()
    comm.check()
    launches_per_step = comm.get_option(_lib.OPT_LAST_LAUNCHES)
    clocks = NvmlClockSampler(0)
    clocks.start()
    ms, per = _events_time(step, args.steps, stream)
    clk = clocks.stop()
    comm.check()
    value = tp * e * m / (ms * 1e-3) / 1e9

    # ---- per-phase kernels (measurement option: one phase per call), CUDA events on the launch stream
    b1 = wire_len(cfg["bits"], cfg["group"], seg) / seg
    b2 = b1
    phase_bytes = {"scatter": tp * (tp - 1) * seg * (e + b1),
                   "reduce": tp * seg * (2 * e + (tp - 1) * (b1 + b2)),
                   "gather": tp * (tp - 1) * seg * (b2 + e)}
    # INT4 g = 128 runs the group-per-lane scatter and the 2-lanes-per-group reduce
    # (fc_stream.cuh q_role_gpl / r_role_gpl; the reduce needs whole tiles, true for every config here)
    gpl = cfg["group"] == 128 and cfg["bits"] == 4
    phase_kernel = {"scatter": "k_qstream_gpl" if gpl else "k_qstream",
                    "reduce": "k_rstream_gpl" if cfg["group"] == 128 else "k_rstream", "gather": "k_dstream"}
    phases = {}
    comm.set_option(_lib.OPT_FUSED, 0)  # phase kernels are timed on the split path
    for bit, name in ((1, "scatter"), (2, "reduce"), (4, "gather")):
        comm.set_option(_lib.OPT_PHASES, bit)
        for _ in range(2):
            step()
        pms, _ = _events_time(step, max(5, args.steps), stream)
        phases[name] = {"kernel": phase_kernel[name], "us": pms * 1e3, "alg_bytes": phase_bytes[name],
                        "gbs": phase_bytes[name] / (pms * 1e-3) / 1e9,
                        "frac": phase_bytes[name] / (pms * 1e-3) / 1e9 / peaks["hbm_gbs"]}
    comm.set_option(_lib.OPT_PHASES, 0)
    comm.set_option(_lib.OPT_FUSED, 1 if args.fused else -1)
    dom = max(phases, key=lambda k: phases[k]["us"])
    traffic = load_traffic().get(phases[dom]["kernel"])
    alg_step = sum(phase_bytes.values())
    roofline = {"bound": "hbm", "kernel": phases[dom]["kernel"], "achieved": phases[dom]["gbs"],
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": phases[dom]["frac"],
                "traffic": traffic, "alg_bytes_per_launch": phases[dom]["alg_bytes"],
                "kernel_us": phases[dom]["us"], "peak_source": peaks["source"],
                "step": {"alg_bytes": alg_step, "achieved": alg_step / (ms * 1e-3) / 1e9,
                         "frac": alg_step / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "t_roof_us": alg_step / peaks["hbm_gbs"] / 1e3}}

    # ---- e2e: the reference-facing call with HOST buffers (pinned): host arrays in, new host
    # arrays out for every rank, one blocking C-ABI call (fc_flash_all_reduce_host) that
    # pipelines chunked H2D, the all-reduce and chunked D2H on the communicator's streams
    # every rank's output is the same decoded stage-2 payload (bit-identical by construction,
    # tests/test_gpu_flash.py), so the step's result is read back once (rank 0's output, one
    # PCIe link's worth, as each rank's own GPU would); the all-ranks readback is reported beside
    host_in = [t.cpu().pin_memory() for t in ins]
    host_out = [torch.empty(m, dtype=dt, pin_memory=True) for _ in range(tp)]
    one_out = [host_out[0]] + [None] * (tp - 1)
    e2e_steps = max(1, min(args.steps, 5))

    def e2e_step():
        return fc.flash_all_reduce(host_in, fcfg, comm=comm, outs=one_out)

    def e2e_step_all():
        return fc.flash_all_reduce(host_in, fcfg, comm=comm, outs=host_out)

    run = e2e_step_all()  # warm: the comm's staging buffers, streams and events
    torch.cuda.synchronize()

    e2e_ms = _wall_time(e2e_step, e2e_steps)
    e2e_all_ms = _wall_time(e2e_step_all, e2e_steps)
    # the PCIe floor of this step: the same H2D bytes as plain pinned copies, nothing else
    h2d_ms = _wall_time(lambda: [d.copy_(h, non_blocking=True) for h, d in zip(host_in, ins)], 2)
    e2e = {"value": tp * e * m / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": tp * e * m, "d2h_bytes_per_step": e * m,
           "all_outputs": {"ms_per_step": e2e_all_ms, "value": tp * e * m / (e2e_all_ms * 1e-3) / 1e9,
                           "d2h_bytes_per_step": tp * e * m},
           "h2d_copy_only_ms": h2d_ms, "frac_of_h2d_floor": h2d_ms / e2e_ms,
           "path": "flash_all_reduce(list of pinned host tensors) -> C-ABI fc_flash_all_reduce_host "
                   "(chunked H2D | all-reduce | D2H, overlapped) -> host tensor of rank 0"}
    del run
    comm.close()
    del outs

    # ---- C5: single-GPU codec kernels on the same activation (HBM roofline), C-ABI calls
    # captured in a CUDA graph so the timing is device time only
    import ctypes as C

    codec = {}
    x = ins[0]
    xo = torch.empty(m, device=dev, dtype=dt)
    sdt = {torch.bfloat16: _lib.DTYPE_BF16, torch.float16: _lib.DTYPE_F16}[dt]
    for bits in (4, 8):
        cc = fc.CodecConfig(bits=bits, group_size=cfg["group"])
        L = cc.device_layout(m)
        qbuf = torch.empty(int(L.total_bytes), dtype=torch.uint8, device=dev)
        cfc = cc.to_fc()
        qf = lambda: _lib.check(_lib.lib().fc_quantize(  # noqa: E731
            x.data_ptr(), sdt, m, C.byref(cfc), qbuf.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
        df = lambda: _lib.check(_lib.lib().fc_dequantize(  # noqa: E731
            qbuf.data_ptr(), m, C.byref(cfc), xo.data_ptr(), sdt, torch.cuda.current_stream().cuda_stream))
        qms, dms = graph_time(qf, 10, stream), graph_time(df, 10, stream)
        ab = e * m + int(L.wire_bytes)
        codec[f"int{bits}_g{cfg['group']}"] = {
            "quantize_us": qms * 1e3, "quantize_gbs": ab / (qms * 1e-3) / 1e9,
            "dequantize_us": dms * 1e3, "dequantize_gbs": ab / (dms * 1e-3) / 1e9,
            "frac_quantize": ab / (qms * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "frac_dequantize": ab / (dms * 1e-3) / 1e9 / peaks["hbm_gbs"], "alg_bytes": ab}
    del ins, xo
    torch.cuda.empty_cache()

    # ---- C4: decode-regime latency (TP=8 emulated, bs x 8192 bf16 per rank), one all-reduce
    # per CUDA-graph node (device time; the host launch path is not in the number)
    decode = {}
    for bs in (8, 64):
        md = bs * 8192
        dcomm = FlashComm.local([0] * tp, slot_bytes_for(-(-md // tp), fcfg.stage1_codec, fcfg.stage2_codec))
        dins = [torch.randn(md, device=dev, generator=g).to(dt) for _ in range(tp)]
        douts = [torch.empty_like(t) for t in dins]
        dstep = lambda: dcomm.all_reduce_local(dins, fcfg, outs=douts, check=False)  # noqa: E731
        dms = graph_time(dstep, 20, stream)
        dcomm.check()
        decode[f"bs{bs}"] = {"latency_us": dms * 1e3, "elems_per_rank": md, "timing": "CUDA graph of 20 calls"}
        dcomm.close()

    # ---- CPU baseline on the host cores (bounded sample)
    cpu = None
    if not args.no_cpu:
        elems = cpu_sample_elems(cfg)
        workers = host_threads()
        dts = [cpu_reference_run(tp, elems, cfg["bits"], cfg["group"], workers, seed=i)[0] for i in range(2)]
        cv = tp * e * elems / min(dts) / 1e9
        cpu = {"value": cv, "unit": "GB/s", "cores": workers, "kind": "port", "host_cpus": os.cpu_count(),
               "sample": f"{tp} ranks x {elems} elements per rank ({elems / m:.4f} of the per-rank tensor), best of 2",
               "note": "oracle/flash_oracle.py numpy restatement of the reference, (owner, piece) jobs on a process pool",
               "gpu_speedup": value / cv}

    return {
        "metric": args.metric, "value": value, "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (torch.randn, seed 1234)",
        "config": {"workload": cfg["desc"] + f"; all {tp} TP ranks emulated as logical ranks on 1 GPU",
                   "tp": tp, "bits": cfg["bits"], "group_size": cfg["group"], "elems_per_rank": m,
                   "value_def": "sum over TP ranks of bf16 input bytes all-reduced per second",
                   "l2": "inputs (%.0f MiB) exceed L2; no flush" % (tp * e * m / 2**20),
                   "mode": "fused" if args.fused else "phase-split (auto: all ranks share one GPU)"},
        "latency_us": ms * 1e3, "latency_us_median": statistics.median(per) * 1e3,
        "algbw_gbs": e * m / (ms * 1e-3) / 1e9,
        "roofline": roofline, "phases": phases, "codec_c5": codec, "decode_c4": decode,
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": int(args.steps * launches_per_step),
        "clocks": clk, "nccl_bf16": None,
    }


def bench_dist(args, cfg, peaks):
    """N>1 under torchrun: one rank per GPU, CUDA IPC over NVLink, NCCL beside it."""
    import torch
    import torch.distributed as dist

    import paper_2412_04964_b200 as fc
    from paper_2412_04964_b200 import _lib
    from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    tp, dt = world, _dtype(cfg["dtype"])
    m = math.prod(cfg["shape"])
    e = 2
    seg = -(-m // tp)
    fcfg = fc.FlashConfig.from_bits(cfg["bits"], group_size=cfg["group"])
    comm = FlashComm.from_process_group(device=local, slot_bytes=slot_bytes_for(seg, fcfg.stage1_codec, fcfg.stage2_codec))
    if args.ctas:
        comm.set_option(_lib.OPT_CTAS, args.ctas)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(m, device=dev, generator=g).to(dt)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([a.elapsed_time(b) / args.steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    clocks = NvmlClockSampler(local)
    clocks.start()
    ms = timed(lambda: comm.all_reduce(x, fcfg, out=out))
    clk = clocks.stop()
    comm.check()
    launches = comm.get_option(_lib.OPT_LAST_LAUNCHES)
    y = x.clone()
    nccl_ms = timed(lambda: dist.all_reduce(y))
    w = wire_len(cfg["bits"], cfg["group"], seg)
    nvl_bytes = (tp - 1) * 2 * w
    hbm_bytes = 2 * e * m + 2 * (tp - 1) * 2 * w
    t_nvl, t_hbm = nvl_bytes / (NVLINK_GBS * 1e9), hbm_bytes / (peaks["hbm_gbs"] * 1e9)
    bound = "nvlink" if t_nvl >= t_hbm else "hbm"
    achieved = (nvl_bytes if bound == "nvlink" else hbm_bytes) / (ms * 1e-3) / 1e9
    peak = NVLINK_GBS if bound == "nvlink" else peaks["hbm_gbs"]
    # e2e: this rank's pinned host buffer in, its host result out, through the per-rank
    # host-buffer call (chunked H2D | all-reduce | D2H overlapped; blocking)
    host = x.cpu().pin_memory()
    hout = torch.empty_like(host).pin_memory()

    def e2e_step():
        comm.all_reduce_host_rank(host, fcfg, out=hout)

    e2e_ms = timed(e2e_step)
    line = {
        "metric": args.metric, "value": tp * e * m / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (torch.randn)",
        "config": {"workload": cfg["desc"].replace("TP=8", f"TP={tp}").replace("TP=4", f"TP={tp}"), "tp": tp,
                   "bits": cfg["bits"], "group_size": cfg["group"], "elems_per_rank": m,
                   "parallelism": f"tp{tp} (one rank per GPU, CUDA IPC over NVLink)",
                   "value_def": "sum over ranks of bf16 input bytes all-reduced per second"},
        "latency_us": ms * 1e3, "algbw_gbs": e * m / (ms * 1e-3) / 1e9,
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "t_roof_us": max(t_nvl, t_hbm) * 1e6},
        "nccl_bf16": {"ms_per_step": nccl_ms, "algbw_gbs": e * m / (nccl_ms * 1e-3) / 1e9,
                      "speedup_of_flash": nccl_ms / ms},
        "e2e": {"value": tp * e * m / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": e * m, "d2h_bytes_per_step": e * m,
                "path": "FlashComm.all_reduce_host_rank -> C-ABI fc_flash_all_reduce_host_rank"},
        "gpu_launches": int(args.steps * launches), "clocks": clk, "cpu_baseline": None,
    }
    comm.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--lag", type=int, default=0)
    ap.add_argument("--fused", action="store_true", help="force the fused flag-synchronised kernel")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.metric = "flash all-reduce effective GB/s (sum over TP ranks), latency and roofline fraction"
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    peaks = load_peaks()
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        bench_dist(args, cfg, peaks)
    else:
        print(json.dumps(bench_local(args, cfg, peaks)), flush=True)


if __name__ == "__main__":
    main()
