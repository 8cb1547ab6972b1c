"""C4 decode-regime latency probe: one-shot cooperative kernel vs the three
streaming kernels, CUDA-graph device time, TP=8 emulated on one GPU."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
from bench import graph_time

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
cfg = fc.FlashConfig.from_bits(4)
for tp in (8,):
    for bs in (1, 8, 16, 32, 64):
        m = bs * 8192
        comm = FlashComm.local([0] * tp, slot_bytes_for(-(-m // tp), cfg.stage1_codec, cfg.stage2_codec))
        ins = [torch.randn(m, device=dev).to(torch.bfloat16) for _ in range(tp)]
        outs = [torch.empty_like(t) for t in ins]
        res = {}
        for name, opts in (("small", {_lib.OPT_ONESHOT: 2}), ("split", {_lib.OPT_ONESHOT: 0}),
                           ("fused", {_lib.OPT_FUSED: 1})):
            comm.set_option(_lib.OPT_ONESHOT, 1)
            comm.set_option(_lib.OPT_FUSED, -1)
            for k, v in opts.items():
                comm.set_option(k, v)
            res[name] = graph_time(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), 20, stream) * 1e3
            comm.check()
            if name == "small":  # eager: host call + launch, CUDA events around 20 calls
                import time
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(20):
                    comm.all_reduce_local(ins, cfg, outs=outs, check=False)
                torch.cuda.synchronize()
                res["small_eager_wall"] = (time.perf_counter() - t0) / 20 * 1e6
        comm.set_option(_lib.OPT_ONESHOT, 0)
        comm.set_option(_lib.OPT_FUSED, -1)
        for ph, name in ((1, "scatter"), (2, "reduce"), (4, "gather")):
            comm.set_option(_lib.OPT_PHASES, ph)
            res[name] = graph_time(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), 20, stream) * 1e3
        comm.set_option(_lib.OPT_PHASES, 2)
        comm.set_option(_lib.OPT_STREAM_MASK, 128)
        res["reduce_lanes32"] = graph_time(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), 20, stream) * 1e3
        comm.set_option(_lib.OPT_PHASES, 1)
        comm.set_option(_lib.OPT_STREAM_MASK, 64)
        res["scatter_lanes32"] = graph_time(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), 20, stream) * 1e3
        comm.set_option(_lib.OPT_STREAM_MASK, 0)
        comm.set_option(_lib.OPT_PHASES, 0)
        comm.close()
        print(json.dumps({"tp": tp, "bs": bs, "latency_us": {k: round(v, 2) for k, v in res.items()}}), flush=True)
x = torch.zeros(1, device=dev)
print(json.dumps({"empty_kernel_in_graph_us": round(graph_time(lambda: x.add_(1), 20, stream) * 1e3, 2)}))
