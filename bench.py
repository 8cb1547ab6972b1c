"""Benchmark of the B200 Flash All-Reduce (BASELINE.json metric:
"all-reduce latency & effective GB/s at TP=2/4/8 vs NCCL bf16; roofline
fraction").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1|c4]

N=1 (the driver default): the headline workload C2 — INT4 asym g128 flash
all-reduce of bf16 [8,1024,8192] per rank at TP=8 — with all 8 TP ranks
emulated on one B200 (8 logical ranks, the reference's list-of-tensors call;
peer stores land in local HBM instead of crossing NVLink). One step = one
all-reduce of all 8 ranks' tensors = three launches (scatter k_qstream_gpl,
reduce k_rstream_gpl, gather k_dstream, launched with programmatic dependent
launch); the fused single-launch kernel is timed beside it, and the same K
steps replayed from one CUDA graph (`roofline.step.ms_graph`: no per-call host
cost) beside the eager `value`.

N>1: one process per GPU (the driver's torchrun launch; `--gpus N` outside
torchrun re-executes itself under torch.distributed.run), TP = N, CUDA IPC
peer buffers over NVLink, the fused kernel k_fstream, NCCL bf16 all_reduce of
the same tensor timed in the same run, and a message-size sweep.

value = sum over TP ranks of the bf16 input bytes all-reduced per second
(whole job); algbw (nccl-tests convention, e*M/t) and latency are reported
too. Inputs (1 GiB at N=1, 128 MiB per GPU at N>1) exceed the 126 MB L2, so no
flush is needed.
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
from typing import Optional

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
# CPU baseline / reference arm: the UNMODIFIED reference (qcollectives, pure
# Python + numpy) installed into baseline/_ref by
#   pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>
# (git-ignored, travels to the GPU box with the snapshot). Its public call
# flash_all_reduce(list of N arrays, FlashConfig) (collectives.py:321-402) runs
# as shipped: one Python thread per rank over the in-process fabric
# (fabric.py:207-217). To use every host core, a pool of processes each runs
# that call on its own token slice of the workload (owners' segments and
# tokens are independent, so the pool's total work equals one call over the
# concatenated slices). Without baseline/_ref the oracle port (test
# infrastructure restating the same algorithm) runs instead, kind "port".

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
HIDDEN = 8192
_REF = {}


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "qcollectives"))


def _bf16_round(x):
    """float32 -> nearest-even bf16 value, kept as float32 (the bf16 activation)."""
    import numpy as np

    u = x.astype(np.float32).view(np.uint32)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.view(np.float32)


def _ref_init(kind, tp, tokens, bits, group, dtype, pin=True):
    """Pool initializer: import the implementation and build this worker's
    inputs once (the reference's own generator, workload.py:111-120)."""
    import multiprocessing as mp

    import numpy as np

    # one core per worker (the reference's rank threads share one GIL; pinned to
    # one core it runs faster than spread over several: one_call_taskset_c0_s)
    ident = getattr(mp.current_process(), "_identity", ())
    if ident and pin:
        try:
            cores = sorted(os.sched_getaffinity(0))
            os.sched_setaffinity(0, {cores[(ident[-1] - 1) % len(cores)]})
        except Exception:
            pass
    _REF.update(kind=kind, tp=tp, tokens=tokens, bits=bits, group=group, xs={})
    if kind == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import qcollectives as q

        _REF["q"] = q
        _REF["cfg"] = q.FlashConfig.from_bits(bits, group_size=group)
    else:
        from oracle import flash_oracle as orc

        _REF["orc"] = orc
        _REF["codec"] = orc.Codec(bits=bits, group_size=group)
    _REF["cast"] = _bf16_round if dtype == "bf16" else (lambda a: a.astype(np.float16).astype(np.float32))


def _ref_inputs(seed):
    xs = _REF["xs"].get(seed)
    if xs is None:
        if _REF["kind"] == "reference":
            q = _REF["q"]
            prof = q.ActivationProfile(hidden_dim=HIDDEN, tokens=_REF["tokens"], seed=seed)
            xs = [_REF["cast"](x) for x in q.gen_rank_activations(prof, _REF["tp"])]
        else:
            orc = _REF["orc"]
            xs = [_REF["cast"](x) for x in orc.gen_rank_activations(HIDDEN, _REF["tokens"], seed, _REF["tp"])]
        _REF["xs"] = {seed: xs}
    return xs


def _ref_prepare(seed):
    _ref_inputs(seed)
    return os.getpid()


def _ref_call(seed):
    """One flash all-reduce of this worker's slice; returns (seconds, checksum)."""
    xs = _ref_inputs(seed)
    t0 = time.perf_counter()
    if _REF["kind"] == "reference":
        run = _REF["q"].flash_all_reduce(xs, _REF["cfg"], timeout=600.0)
        out = run.outputs[0]
    else:
        out = _REF["orc"].flash_all_reduce(xs, _REF["codec"], _REF["codec"]).outputs[0]
    dt = time.perf_counter() - t0
    return dt, float(out.ravel()[::4099].astype("float64").sum())


def _pinned_call(args):
    """One as-shipped call in a fresh process pinned to core 0 (taskset -c 0)."""
    kind, tp, tokens, bits, group, dtype, seed = args
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    _ref_init(kind, tp, tokens, bits, group, dtype, pin=False)
    return _ref_call(seed)[0]


class CpuReference:
    """A persistent pool of `workers` processes, each owning a slice of
    `tokens` tokens x 8192 per rank; one step = every worker runs one
    flash_all_reduce on its slice concurrently."""

    def __init__(self, cfg: dict, workers: int, tokens: int, kind: Optional[str] = None):
        import multiprocessing as mp

        self.kind = kind or ("reference" if have_reference() else "port")
        self.cfg, self.workers, self.tokens = cfg, workers, tokens
        self.init = (self.kind, cfg["tp"], tokens, cfg["bits"], cfg["group"], cfg["dtype"])
        self.pool = mp.get_context("fork").Pool(workers, initializer=_ref_init, initargs=self.init)
        self.elems_per_rank = workers * tokens * HIDDEN

    def step(self, seed: int) -> float:
        seeds = [seed * 1000 + w for w in range(self.workers)]
        self.pool.map(_ref_prepare, seeds, chunksize=1)  # inputs built outside the timed region
        t0 = time.perf_counter()
        res = self.pool.map(_ref_call, seeds, chunksize=1)
        wall = time.perf_counter() - t0
        self.last_call_s = statistics.mean(r[0] for r in res)
        return wall

    def gbs(self, seconds: float) -> float:
        return self.cfg["tp"] * 2 * self.elems_per_rank / seconds / 1e9

    def as_shipped(self, seed: int = 7) -> dict:
        """One call of one slice in one process, unpinned and pinned to one core."""
        import multiprocessing as mp

        with mp.get_context("fork").Pool(1, initializer=_ref_init, initargs=self.init + (False,)) as p:
            free_s = p.apply(_ref_call, (seed,))[0]
        with mp.get_context("fork").Pool(1) as p:
            pinned_s = p.apply(_pinned_call, (self.init + (seed,),))
        return {"elements_per_rank": self.tokens * HIDDEN, "one_call_s": free_s, "one_call_taskset_c0_s": pinned_s,
                "one_call_gbs": self.gbs(free_s) / self.workers,
                "one_call_taskset_c0_gbs": self.gbs(pinned_s) / self.workers}

    def describe(self) -> str:
        what = ("unmodified qcollectives.flash_all_reduce from baseline/_ref (thread per rank, as shipped; "
                "each pool process pinned to its own core)"
                if self.kind == "reference" else "oracle/flash_oracle.py port of qcollectives.flash_all_reduce")
        return (f"{what}; {self.workers} processes x one call each on {self.tokens} tokens x {HIDDEN} per rank "
                f"({self.cfg['tp']} ranks, {self.cfg['dtype']}-valued float32 arrays from the reference's "
                f"gen_rank_activations) = {self.elems_per_rank} elements per rank per step "
                f"({self.elems_per_rank / math.prod(self.cfg['shape']):.4f} of the per-rank tensor)")

    def close(self):
        self.pool.terminate()
        self.pool.join()


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_tokens(cfg: dict, workers: int, frac: float) -> int:
    """Tokens per worker slice so the pool covers about `frac` of the per-rank tensor."""
    tokens = math.prod(cfg["shape"]) // HIDDEN
    return max(1, int(tokens * frac) // workers)


def run_reference(args, cfg):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    workers = host_threads()
    # about 1/8 of the per-rank tensor per step at C2 (the whole call takes ~55 s on one core)
    ref = CpuReference(cfg, workers, ref_tokens(cfg, workers, 1.0 / 8 if cfg["tp"] >= 8 else 1.0 / 2))
    try:
        times = []
        for i in range(args.warmup + args.steps):
            dt = ref.step(i)
            if i >= args.warmup:
                times.append(dt)
        shipped = ref.as_shipped()
    finally:
        ref.close()
    t = statistics.mean(times)
    val = ref.gbs(t)
    sample = ref.describe()
    line = {"impl": "reference", "metric": args.metric, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (numpy)", "data": "synthetic",
            "config": {"workload": cfg["desc"], "tp": cfg["tp"], "sample": sample},
            "cpu_baseline": {"value": val, "unit": "GB/s", "cores": workers, "kind": ref.kind, "sample": sample,
                             "host_cpus": os.cpu_count(), "as_shipped": shipped},
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


def load_traffic(config: str) -> dict:
    """ncu DRAM bytes (read + write) per launch, keyed by bench config then kernel
    (profiles/ncu_traffic.json, written by tools/make_traffic.py from one
    `ncu --set full` capture of that config)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d.get(config, {}) if isinstance(d.get(config), dict) else {}
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
    # beside (not the value): the same K steps captured in one CUDA graph, as a serving engine
    # replays them -- no per-call host launch cost (it bounds the small C1 / C4 steps)
    gms = graph_time(step, args.steps, stream)
    comm.check()

    # ---- per-phase kernels (measurement option: one phase per call), CUDA events on the launch stream
    b1 = wire_len(cfg["bits"], cfg["group"], seg) / seg
    b2 = b1
    # g = 128 (one storage width) runs the 2-lanes-per-group reduce, which reads every source
    # piece from the receive slots, the own one too: the scatter then also quantizes the own
    # piece (ownq, fc_stream.cuh r_role_gpl). Per-phase bytes are what each kernel must move;
    # the step's algorithmic bytes stay the minimum (own piece kept on chip), so
    # the ownq detour (+2 b1 per own element) counts against the step fraction
    ownq = 1 if cfg["group"] == 128 else 0
    phase_bytes = {"scatter": tp * (tp - 1 + ownq) * seg * (e + b1),
                   "reduce": tp * seg * ((tp - 1 + ownq) * b1 + (1 - ownq) * e + (tp - 1) * b2 + e),
                   "gather": tp * (tp - 1) * seg * (b2 + e)}
    # per rank: input read + output write (2 e M) + the N-1 peer pieces of both stages written and read once
    alg_step = tp * (2 * e * m + 2 * (tp - 1) * seg * (b1 + b2))
    # INT4 g = 128 runs the group-per-lane scatter (q_role_gpl)
    # (INT8 too for rounds up to 256 tiles per segment, fc_run.cuh launch_qstream)
    gpl = cfg["group"] == 128 and (cfg["bits"] == 4 or seg <= 256 * 8192)
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
    # the single-launch fused kernel (k_fstream, the cross-GPU default) on the same workload
    comm.set_option(_lib.OPT_FUSED, 1)
    for _ in range(2):
        step()
    fms, _ = _events_time(step, max(5, args.steps), stream)
    comm.check()
    fused = {"kernel": "k_fstream", "ms_per_step": fms, "launches_per_step": comm.get_option(_lib.OPT_LAST_LAUNCHES),
             "vs_split": fms / ms}
    comm.set_option(_lib.OPT_FUSED, 1 if args.fused else -1)
    dom = max(phases, key=lambda k: phases[k]["us"])
    traffic = load_traffic(args.config).get(phases[dom]["kernel"])
    roofline = {"bound": "hbm", "kernel": phases[dom]["kernel"], "achieved": phases[dom]["gbs"],
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": phases[dom]["frac"],
                "traffic": traffic, "alg_bytes_per_launch": phases[dom]["alg_bytes"],
                "kernel_us": phases[dom]["us"], "peak_source": peaks["source"],
                "step": {"alg_bytes": alg_step, "achieved": alg_step / (ms * 1e-3) / 1e9,
                         "frac": alg_step / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "t_roof_us": alg_step / peaks["hbm_gbs"] / 1e3,
                         "ms_graph": gms, "frac_graph": alg_step / (gms * 1e-3) / 1e9 / peaks["hbm_gbs"]}}

    # ---- e2e: the reference-facing call with HOST buffers (pinned): every rank's host array
    # in, a new host array out for EVERY rank (the reference returns all N outputs), one
    # blocking C-ABI call (fc_flash_all_reduce_host) that pipelines chunked H2D, the
    # all-reduce and chunked D2H on the communicator's streams
    host_in = [t.cpu().pin_memory() for t in ins]
    host_out = [torch.empty(m, dtype=dt, pin_memory=True) for _ in range(tp)]
    one_out = [host_out[0]] + [None] * (tp - 1)
    e2e_steps = max(1, min(args.steps, 5))

    def e2e_step_all():
        return fc.flash_all_reduce(host_in, fcfg, comm=comm, outs=host_out)

    def e2e_step_one():
        return fc.flash_all_reduce(host_in, fcfg, comm=comm, outs=one_out)

    run = e2e_step_all()  # warm: the comm's staging buffers, streams and events
    torch.cuda.synchronize()

    e2e_ms = _wall_time(e2e_step_all, e2e_steps)
    e2e_one_ms = _wall_time(e2e_step_one, e2e_steps)
    # the PCIe floor of this step: the same H2D + D2H bytes as plain pinned copies, nothing else
    h2d_ms = _wall_time(lambda: [d.copy_(h, non_blocking=True) for h, d in zip(host_in, ins)], 2)
    d2h_ms = _wall_time(lambda: [h.copy_(d, non_blocking=True) for h, d in zip(host_out, ins)], 2)
    e2e = {"value": tp * e * m / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": tp * e * m, "d2h_bytes_per_step": tp * e * m,
           "rank0_output_only": {"ms_per_step": e2e_one_ms, "value": tp * e * m / (e2e_one_ms * 1e-3) / 1e9,
                                 "d2h_bytes_per_step": e * m},
           "h2d_copy_only_ms": h2d_ms, "d2h_copy_only_ms": d2h_ms,
           "path": "flash_all_reduce(list of pinned host tensors) -> C-ABI fc_flash_all_reduce_host "
                   "(chunked H2D | all-reduce | D2H, overlapped) -> a host tensor for every rank"}
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
    for bits, grp in [(b, g_) for b in (4, 8) for g_ in (32, 64, 128, 256)] + [("e4m3", 128), ("e2m1", 128)]:
        cc = fc.CodecConfig(bits=bits, group_size=grp) if isinstance(bits, int) else \
            fc.CodecConfig(number_format=bits, group_size=grp)
        L = cc.device_layout(m)
        qbuf = torch.empty(int(L.total_bytes), dtype=torch.uint8, device=dev)
        cfc = cc.to_fc()
        qf = lambda: _lib.check(_lib.lib().fc_quantize(  # noqa: E731
            x.data_ptr(), sdt, m, C.byref(cfc), qbuf.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
        df = lambda: _lib.check(_lib.lib().fc_dequantize(  # noqa: E731
            qbuf.data_ptr(), m, C.byref(cfc), xo.data_ptr(), sdt, torch.cuda.current_stream().cuda_stream))
        qms, dms = graph_time(qf, 10, stream), graph_time(df, 10, stream)
        ab = e * m + int(L.wire_bytes)
        codec[(f"int{bits}" if isinstance(bits, int) else bits) + f"_g{grp}"] = {
            "quantize_us": qms * 1e3, "quantize_gbs": ab / (qms * 1e-3) / 1e9,
            "dequantize_us": dms * 1e3, "dequantize_gbs": ab / (dms * 1e-3) / 1e9,
            "frac_quantize": ab / (qms * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "frac_dequantize": ab / (dms * 1e-3) / 1e9 / peaks["hbm_gbs"], "alg_bytes": ab}
    # ---- minifloat and rotated flash on the C2 workload, 8 logical ranks on this GPU, three
    # launches per step: e4m3 stage codecs (cvt.rn.satfinite) on the TMA-fed streaming kernels
    # (MfSpec) and, beside, on the lane-8 kernels (fc_l8.cuh, FC_OPT_STREAM_MASK bit 10); INT4
    # g128 with the Hadamard rotation (block 128, seeded signs) fused into the lane-8 kernels'
    # prologue / epilogue
    lane8 = {}
    e4 = fc.FlashConfig.uniform(fc.CodecConfig(number_format="e4m3"))
    for name, lcfg, lmask, kern in (
            ("e4m3_g128", e4, 0, "k_qstream_gpl | k_rstream_gpl | k_dstream <MfSpec e4m3>"),
            ("e4m3_g128_lane8", e4, 1024, "k_l8_scatter | k_l8_reduce | k_l8_gather"),
            ("int4_g128_rot128", fc.FlashConfig(fc.CodecConfig(bits=4), fc.CodecConfig(bits=4),
                                                rotation=fc.HadamardBlock(128, sign_seed=1)), 0,
             "k_l8_scatter | k_l8_reduce | k_l8_gather")):
        lcomm = FlashComm.local([0] * tp, slot_bytes_for(seg, lcfg.stage1_codec, lcfg.stage2_codec))
        if lmask:
            lcomm.set_option(_lib.OPT_STREAM_MASK, lmask)
        louts = [torch.empty(m, device=dev, dtype=dt) for _ in range(tp)]
        signs = None
        if lcfg.rotation is not None:
            signs = [lcfg.rotation._device_signs(dev) for _ in range(tp)]
            lcomm.set_rotation(lcfg.rotation, signs)
        lstep = lambda: lcomm.all_reduce_local(ins, lcfg, outs=louts, check=False)  # noqa: E731
        for _ in range(3):
            lstep()
        lcomm.check()
        lms, _ = _events_time(lstep, max(5, args.steps // 2), stream)
        lcomm.check()
        b1l = lcfg.stage1_codec.device_layout(seg).wire_bytes / seg
        lb = tp * (2 * e * m + 2 * (tp - 1) * seg * 2 * b1l)
        lane8[name] = {"ms_per_step": lms, "value_gbs": tp * e * m / (lms * 1e-3) / 1e9,
                       "hbm_alg_bytes": lb, "frac": lb / (lms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                       "launches_per_step": lcomm.get_option(_lib.OPT_LAST_LAUNCHES),
                       "kernels": kern}
        lcomm.set_rotation(None)
        lcomm.close()
        del louts, signs
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

    # ---- CPU baseline on the host cores (bounded sample): the unmodified reference (baseline/_ref)
    cpu = None
    if not args.no_cpu:
        workers = host_threads()
        ref = CpuReference(cfg, workers, ref_tokens(cfg, workers, 1.0 / 8))
        try:
            ref.step(0)  # warm (imports, page faults)
            dts = [ref.step(i) for i in (1, 2)]
        finally:
            ref.close()
        cv = ref.gbs(min(dts))
        cpu = {"value": cv, "unit": "GB/s", "cores": workers, "kind": ref.kind, "host_cpus": os.cpu_count(),
               "sample": ref.describe() + ", best of 2 steps", "gpu_speedup": value / cv,
               "e2e_speedup": e2e["value"] / cv}

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
        "roofline": roofline, "phases": phases, "fused_one_gpu": fused, "codec_c5": codec, "decode_c4": decode,
        "lane8": lane8,
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": int(args.steps * launches_per_step),
        "clocks": clk, "nccl_bf16": None,
    }


NVLINK_NOMINAL_GBS = 900.0  # per direction per GPU (north_star roofline)
NVLINK_MEASURED_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def dist_roofline(tp: int, m: int, e: int, w1: int, w2: int, hbm_gbs: float, ms: float) -> dict:
    """Per-rank roofline of one all-reduce: NVLink bytes per
    direction (N-1)(w1 + w2) (the reference's _flash_wire_bytes,
    costmodel.py:122-128) at 900 GB/s, HBM bytes 2eM + 2(N-1)(w1 + w2) at the
    measured copy peak; the slower bounds."""
    nvl = (tp - 1) * (w1 + w2)
    hbm = 2 * e * m + 2 * (tp - 1) * (w1 + w2)
    t_nvl, t_hbm = nvl / (NVLINK_NOMINAL_GBS * 1e9), hbm / (hbm_gbs * 1e9)
    bound = "nvlink" if t_nvl >= t_hbm else "hbm"
    alg = nvl if bound == "nvlink" else hbm
    peak = NVLINK_NOMINAL_GBS if bound == "nvlink" else hbm_gbs
    achieved = alg / (ms * 1e-3) / 1e9
    t_meas = max(nvl / (NVLINK_MEASURED_GBS * 1e9), t_hbm)
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "t_roof_us": max(t_nvl, t_hbm) * 1e6, "nvlink_bytes_per_rank": nvl,
            "hbm_bytes_per_rank": hbm, "nvlink_peak_note": "900 GB/s nominal per direction (north_star)",
            "frac_at_measured_770": t_meas * 1e3 / ms}


def bench_dist(args, cfg, peaks):
    """N>1: one rank per GPU, TP = world size, CUDA IPC peer buffers over NVLink
    (fused kernel k_fstream), NCCL bf16 all_reduce of the same tensor beside it.
    FC_BENCH_SHARED_GPU=1 is a one-GPU dry run of this exact code (all ranks on
    cuda:0, gloo for the handle exchange, NCCL leg skipped) for the GPU tests."""
    import torch
    import torch.distributed as dist

    import paper_2412_04964_b200 as fc
    from paper_2412_04964_b200 import _lib
    from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    shared = os.environ.get("FC_BENCH_SHARED_GPU") == "1"
    local = 0 if shared else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    tp, dt = world, _dtype(cfg["dtype"])
    m = math.prod(cfg["shape"])
    e = 2
    seg = -(-m // tp)
    fcfg = fc.FlashConfig.from_bits(cfg["bits"], group_size=cfg["group"])
    sizes = [m] + [b // e for b in (1 << 16, 1 << 20, 1 << 24)]
    slot = max(slot_bytes_for(-(-n // tp), c, c) for n in sizes for c in
               (fc.CodecConfig(bits=4, group_size=cfg["group"]), fc.CodecConfig(bits=8, group_size=cfg["group"])))
    comm = FlashComm.from_process_group(device=local, slot_bytes=slot)
    if args.ctas:
        comm.set_option(_lib.OPT_CTAS, args.ctas)
    if args.fused:
        comm.set_option(_lib.OPT_FUSED, 1)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn(m, device=dev, generator=g).to(dt)
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    def max_over_ranks(v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    def timed(fn, steps=None, warmup=None):
        """ms per call: barrier + synchronize on both sides, CUDA events on the
        launching stream, max over ranks."""
        steps = steps or args.steps
        for _ in range(warmup if warmup is not None else args.warmup):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        return max_over_ranks(a.elapsed_time(b) / steps)

    clocks = NvmlClockSampler(local)
    clocks.start()
    ms = timed(lambda: comm.all_reduce(x, fcfg, out=out))
    clk = clocks.stop()
    comm.check()
    launches = comm.get_option(_lib.OPT_LAST_LAUNCHES)
    w1 = wire_len(cfg["bits"], cfg["group"], seg)
    roof = dist_roofline(tp, m, e, w1, w1, peaks["hbm_gbs"], ms)
    roof["kernel"] = "k_fstream" if launches <= 2 else "phase-split kernels"
    roof["peak_source"] = "nvlink nominal" if roof["bound"] == "nvlink" else peaks["source"]

    # the phase-split path across GPUs (k_qstream_gpl | barrier | k_rstream_gpl | barrier | k_dstream)
    comm.set_option(_lib.OPT_FUSED, 0)
    split_ms = timed(lambda: comm.all_reduce(x, fcfg, out=out))
    comm.set_option(_lib.OPT_FUSED, 1 if args.fused else -1)
    comm.check()

    nccl = None
    if not shared:
        y = x.clone()
        nccl_ms = timed(lambda: dist.all_reduce(y))
        nccl = {"ms_per_step": nccl_ms, "algbw_gbs": e * m / (nccl_ms * 1e-3) / 1e9,
                "busbw_gbs": e * m / (nccl_ms * 1e-3) / 1e9 * 2 * (tp - 1) / tp, "speedup_of_flash": nccl_ms / ms}

    # message-size sweep (C3 subset): flash INT4 / INT8 and NCCL bf16 at the same sizes
    sweep = []
    for n in sorted(set(sizes)):
        xs_ = x[:n]
        os_ = out[:n]
        row = {"bytes": e * n}
        for bits in (4, 8):
            c = fc.FlashConfig.from_bits(bits, group_size=cfg["group"])
            row[f"int{bits}_us"] = timed(lambda: comm.all_reduce(xs_, c, out=os_), steps=max(10, args.steps)) * 1e3
        if not shared:
            ys = x[:n].clone()
            row["nccl_bf16_us"] = timed(lambda: dist.all_reduce(ys), steps=max(10, args.steps)) * 1e3
            row["int4_speedup"] = row["nccl_bf16_us"] / row["int4_us"]
        sweep.append(row)
    comm.check()

    # decode regime (C4): bs x 8192 per rank, eager calls (host launch path included)
    decode = {}
    for bs in (8, 64):
        n = bs * 8192
        xs_, os_ = x[:n], out[:n]
        decode[f"bs{bs}"] = {"latency_us": timed(lambda: comm.all_reduce(xs_, fcfg, out=os_),
                                                 steps=max(20, args.steps)) * 1e3, "timing": "eager calls"}
    comm.check()

    # e2e: this rank's pinned host buffer in, its host result out, through the per-rank
    # host-buffer call (chunked H2D | all-reduce | D2H overlapped; blocking)
    host = x.cpu().pin_memory()
    hout = torch.empty_like(host).pin_memory()
    e2e_ms = timed(lambda: comm.all_reduce_host_rank(host, fcfg, out=hout), steps=max(1, min(args.steps, 5)))
    line = {
        "metric": args.metric, "value": tp * e * m / (ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (torch.randn)",
        "config": {"workload": cfg["desc"].replace("TP=8", f"TP={tp}").replace("TP=4", f"TP={tp}"), "tp": tp,
                   "bits": cfg["bits"], "group_size": cfg["group"], "elems_per_rank": m,
                   "parallelism": f"tp{tp} (one rank per GPU, CUDA IPC over NVLink)" +
                                  (" [dry run: all ranks on cuda:0]" if shared else ""),
                   "value_def": "sum over ranks of bf16 input bytes all-reduced per second",
                   "l2": "inputs (%.0f MiB per GPU) exceed L2; no flush" % (e * m / 2**20)},
        "latency_us": ms * 1e3, "algbw_gbs": e * m / (ms * 1e-3) / 1e9,
        "busbw_gbs": e * m / (ms * 1e-3) / 1e9 * 2 * (tp - 1) / tp,
        "roofline": roof, "split_path_ms": split_ms, "nccl_bf16": nccl, "sweep": sweep, "decode_c4": decode,
        "e2e": {"value": tp * e * m / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": e * m, "d2h_bytes_per_step": e * m,
                "path": "FlashComm.all_reduce_host_rank -> C-ABI fc_flash_all_reduce_host_rank (per rank)"},
        "gpu_launches": int(args.steps * launches), "clocks": clk, "cpu_baseline": None,
    }
    comm.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def reexec_torchrun(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) the
    way the driver does."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if os.environ.get("FC_BENCH_SHARED_GPU") != "1" and have < args.gpus:
        print(json.dumps({"metric": args.metric, "error": f"--gpus {args.gpus} but only {have} GPUs visible"}))
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(reexec_torchrun(args))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        bench_dist(args, cfg, peaks)
    else:
        print(json.dumps(bench_local(args, cfg, peaks)), flush=True)


if __name__ == "__main__":
    main()
