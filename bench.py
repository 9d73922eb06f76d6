#!/usr/bin/env python
"""Benchmark of the memory-layer hot path (arXiv 2412.09764) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5|...] [--per-rank G]

A step is one pass of the whole hot path over one
batch: memory_layer_fwd + memory_layer_bwd (product-key top-k, softmax,
EmbeddingBag fwd with the Memory+ silu gate, gate backward, the sorted
"reverse_indices" EmbeddingBag backward, softmax / key / query backward).

N = 1: BASELINE config[1] (C2: N = 1024^2 values x 2048, 4 heads, k = 32,
16K tokens, bf16).  N > 1 (`--gpus N` re-executes itself under
torch.distributed.run, one rank per GPU, unless WORLD_SIZE is already set):
the dim-sharded memory group of §3.1.2 -- every rank scores its own
tokens, the value table is sharded G ways along the value dim.  c1-c3 keep
16K tokens per rank (weak scaling); c4/c5 (8192^2 keys)
split a fixed global batch over the ranks.

`--per-rank G` runs, on ONE GPU, the per-rank work of the G-rank step with
the collectives replaced by local copies (SURVEY §8(e) t_ref(G)): a1-a4 on
this rank's tokens, the bag forward/backward over all G ranks' tokens on an
[N, dv/G] value shard, the gate on this rank's tokens.  That is how the
8192^2-key configurations (256-512 GiB of values, more than one B200 holds)
are measured on one GPU.  Under N > 1 the same loopback step is also timed
after the real one and E(G) = t_ref(G) / t_G is reported.

Inputs are synthetic (counter-based generator), generated
on the device before timing.  The value table (>= 4 GiB) is > 30x the 126 MB
L2, so no L2 flush is needed between steps ("inputs_larger_than_L2").
Prints ONE JSON line on rank 0.
"""
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
# the caching allocator grows by mapping pages into expandable segments
# instead of cudaMalloc-ing new ones (a 10-200 ms host stall when it happens
# inside a timed step with tens of GB of per-step buffers, C5)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

CONFIGS = {
    # T: tokens per rank (weak scaling); T_global: fixed global batch split over the ranks
    "c1": dict(S=32, dv=64, D=64, Dk=32, H=1, k=4, T=256, dtype="f32",
               desc="tiny PKM: N=1024, d=64, 1 head, k=4, 256 tokens, fp32"),
    "c2": dict(S=1024, dv=2048, D=2048, Dk=1024, H=4, k=32, T=16384, dtype="bf16",
               desc="1.3B-base memory layer: N=1024^2 x 2048, 4 heads, k=32, 16K tokens, bf16"),
    "c3": dict(S=4096, dv=2048, D=2048, Dk=1024, H=4, k=32, T=16384, dtype="bf16",
               desc="N=4096^2 x 2048 bf16, 4 heads, k=32, 16K tokens per rank, dim-sharded"),
    "c4": dict(S=8192, dv=2048, D=2048, Dk=1024, H=4, k=32, T_global=16384, dtype="bf16",
               desc="N=8192^2 x 2048 bf16 (256 GiB of values), gated, 4 heads, k=32, "
                    "16K tokens per step over the group, dim-sharded"),
    "c5": dict(S=8192, dv=4096, D=4096, Dk=2048, H=4, k=32, T_global=65536, dtype="bf16",
               desc="8B-base scale: N=8192^2 x 4096 bf16 (512 GiB of values), 4 heads, k=32, "
                    "64K tokens per step over the group, dim-sharded"),
    # value-dim sweep of the paper's range (north_star: value dims 1024 to 4096), N = 1024^2
    "c2_dv1024": dict(S=1024, dv=1024, D=1024, Dk=1024, H=4, k=32, T=16384, dtype="bf16",
                      desc="N=1024^2 x 1024, 4 heads, k=32, 16K tokens, bf16"),
    "c2_dv4096": dict(S=1024, dv=4096, D=4096, Dk=1024, H=4, k=32, T=16384, dtype="bf16",
                      desc="N=1024^2 x 4096, 4 heads, k=32, 16K tokens, bf16"),
}
METRIC = "memory-layer fwd+bwd tok/s (EmbeddingBag fwd/bwd HBM GB/s, % peak)"
SEED = 0
NVLINK_PEER_GBS = 770.0    # B200_PROFILING.md: measured peer copy per direction (nominal 900)


def tokens_per_rank(cfg, G):
    if "T_global" in cfg:
        if cfg["T_global"] % G:
            raise SystemExit(f"{cfg['name']}: G={G} must divide the global batch {cfg['T_global']}")
        return cfg["T_global"] // G
    return cfg["T"]


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # first queries outside the timed region (the first NVML query of a
            # process can stall the driver for tens of milliseconds)
            for _ in range(3):
                pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS") == "1":
            self.nv = None
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------- dist helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def respawn_under_torchrun(n):
    """`--gpus N` without a torchrun environment: re-execute this command with
    one rank per GPU (rendezvous on 127.0.0.1) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------- comm wrappers
class CGroup:
    """Marks the C-ABI memory group (ops.Group over NCCL) for build_step."""

    def __init__(self, grp):
        self.grp = grp


def coll_bytes(cfg, G, T_loc, mode):
    """Bytes one rank sends over NVLink per step, per collective kind of the
    C-ABI group (include/memlayer.h memory_layer_*_group)."""
    e = 2 if cfg["dtype"] == "bf16" else 4
    B = cfg["H"] * cfg["k"]
    dvG = cfg["dv"] // G
    blk = T_loc * dvG * e
    out = {"nccl_all_gather": (G - 1) * T_loc * 2 * B * 4,         # packed (idx, w)
           "nccl_all_to_all": (G - 1) * blk,                      # dy slices
           "nccl_reduce_scatter": (G - 1) * T_loc * B * 4}        # partial dw
    if mode == "alltoall":
        if os.environ.get("ML_GROUP_PIPELINE") == "1":
            out["nccl_sendrecv"] = (G - 1) * blk                  # the forward's blocks (ring)
        else:
            out["nccl_all_to_all"] += (G - 1) * blk               # the forward's blocks
    else:
        out["nccl_all_gather"] += G * (G - 1) * blk               # every block to everyone
    return out


def coll_report(kern, steps, cfg, G, T_loc, mode):
    nb = coll_bytes(cfg, G, T_loc, mode)
    out = {}
    for kind, b in nb.items():
        if kind not in kern:
            continue
        cnt, tot = kern[kind]
        ms = tot / steps
        gbs = b / (ms / 1e3) / 1e9 if ms > 0 else None
        out[kind] = {"calls_per_step": cnt / steps, "ms_per_step": round(ms, 4),
                     "link_bytes_per_step": b, "GBps": round(gbs, 1) if gbs else None,
                     "frac_of_peer_copy": round(gbs / NVLINK_PEER_GBS, 4) if gbs else None}
    out["note"] = ("per-rank bytes sent over NVLink / collective time (serialised measurement pass); "
                   f"peer-copy reference {NVLINK_PEER_GBS} GB/s per direction (B200_PROFILING.md)")
    return out


# ------------------------------------------------------------- our arm
def synth_value_shard(N, dv, G, rank, dt, dev, ops, torch):
    """This rank's [N, dv/G] column shard of the synthetic value table,
    regenerated from the same counters as the full table (i = r*dv + c)."""
    from synthetic import gen
    lo, hi = rank * dv // G, (rank + 1) * dv // G
    out = torch.empty((N, hi - lo), dtype=dt, device=dev)
    buf = torch.empty((1 << 16, dv), dtype=dt, device=dev)
    for r0 in range(0, N, buf.shape[0]):
        n = min(buf.shape[0], N - r0)
        ops.synth_fill(buf[:n], SEED, gen.TAGS["V"], row0=r0)
        out[r0:r0 + n].copy_(buf[:n, lo:hi])
    del buf
    return out


def make_inputs(cfg, dev, G, rank, ops, torch, sharded):
    from synthetic import gen
    S, dv, D, Dk, H = (cfg[n] for n in ("S", "dv", "D", "Dk", "H"))
    T = tokens_per_rank(cfg, G)
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    N = S * S
    t = {}

    def fill(name, shape, tag, scale=1.0, row0=0, dtype=dt):
        x = torch.empty(shape, dtype=dtype, device=dev)
        ops.synth_fill(x, SEED, gen.TAGS[tag], scale=scale, row0=row0)
        t[name] = x

    T0 = rank * T  # this rank's token rows of the global batch
    fill("q", (T, H, Dk), "q", row0=T0 * H)
    fill("x", (T, D), "x", row0=T0)
    fill("dout", (T, D), "dout", row0=T0)
    fill("K1", (H, S, Dk // 2), "K1", gen.scale_for("K1", Dk=Dk))
    fill("K2", (H, S, Dk // 2), "K2", gen.scale_for("K2", Dk=Dk))
    fill("W1", (D, dv), "W1", gen.scale_for("W1", D=D))
    fill("W2", (dv, D), "W2", gen.scale_for("W2", dv=dv))
    if not sharded:
        fill("V", (N, dv), "V")
    else:
        # this rank's column shard [N, dv/G] of V (regenerated from the same
        # counters as the full table, columns [rank*dv/G, (rank+1)*dv/G))
        t["V"] = synth_value_shard(N, dv, G, rank, dt, dev, ops, torch)
    return t


def group_others(cfg, G, rank, t, ops, torch):
    """The (idx, w) every other rank of a G-rank group would contribute to
    the all-gather, computed on this GPU once before timing (--per-rank)."""
    from synthetic import gen
    H, Dk, k = cfg["H"], cfg["Dk"], cfg["k"]
    T = tokens_per_rank(cfg, G)
    idx_all = torch.empty((G * T, H, k), dtype=torch.int32, device=t["q"].device)
    w_all = torch.empty((G * T, H, k), dtype=torch.float32, device=t["q"].device)
    lists = torch.empty((G, 2, T * H * k), dtype=torch.int32, device=t["q"].device)
    q = torch.empty_like(t["q"])
    for g in range(G):
        ops.synth_fill(q, SEED, gen.TAGS["q"], row0=g * T * H)
        i, w = ops.pkm_topk(q, t["K1"], t["K2"], k)
        idx_all[g * T:(g + 1) * T].copy_(i)
        w_all[g * T:(g + 1) * T].copy_(w)
        # rank g's sorted share of the group's inverse map
        ops.group_sort_local(cfg["S"] ** 2, i.view(T, H * k), g, out=lists[g])
    return {"idx_all": idx_all, "w_all": w_all, "lists": lists}


def loopback_group(G, rank, others, ops, torch):
    """The C-ABI loopback group of one rank (include/memlayer.h
    ml_group_init_loopback) from the other ranks' captured data: the packed
    (idx, w) [G*T_loc, 2B] int32 (w as bits) and the sorted lists."""
    idx_all, w_all = others["idx_all"], others["w_all"]
    n = idx_all.shape[0]
    iw = torch.cat([idx_all.reshape(n, -1), w_all.reshape(n, -1).view(torch.int32)], 1).contiguous()
    return ops.Group.loopback(G, rank, [iw, others["lists"].contiguous()])


def build_step(args, cfg, t, ops, torch, comm=None):
    """One fwd + bwd step through the public API; `comm` selects the memory
    group path (GroupMemoryLayer over that communicator)."""
    k = cfg["k"]
    dK1 = torch.zeros(t["K1"].shape, dtype=torch.float32, device=t["q"].device)
    dK2 = torch.zeros(t["K2"].shape, dtype=torch.float32, device=t["q"].device)
    bufs = {}
    dV_dtype = torch.bfloat16 if args.dv_dtype == "bf16" else torch.float32
    if isinstance(comm, CGroup):
        # the product path for N > 1: the memory group behind the C ABI
        # (exchange, overlap and local kernels inside libmemlayer, NCCL)
        from paper_2412_09764_b200 import group
        layer = group.CGroupMemoryLayer(comm.grp, k=k, mode=args.mode, dV_dtype=dV_dtype)

        def step(inp=t):
            dK1.zero_()
            dK2.zero_()
            out, saved = layer.forward(inp["x"], inp["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"])
            g = layer.backward(inp["dout"], saved, dK1, dK2)
            step.last_saved = saved
            return out, g
    elif comm is not None:
        from paper_2412_09764_b200 import group
        layer = group.GroupMemoryLayer(comm, k=k, mode=args.mode,
                                       local=group.CudaLocal(dV_dtype=dV_dtype))

        def step(inp=t):
            dK1.zero_()
            dK2.zero_()
            out, saved = layer.forward(inp["x"], inp["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"])
            g = layer.backward(inp["dout"], saved, dK1, dK2)
            step.last_saved = saved
            return out, g
    else:
        def step(inp=t):
            dK1.zero_()
            dK2.zero_()
            out, saved = ops.memory_layer_fwd(inp["x"], inp["q"], t["K1"], t["K2"], t["V"],
                                              t["W1"], t["W2"], k, qk_norm=args.qk_norm,
                                              keep_state=not args.no_state)
            g = ops.memory_layer_bwd(inp["dout"], inp["x"], inp["q"], t["K1"], t["K2"], t["V"],
                                     t["W1"], t["W2"], saved, dK1=dK1, dK2=dK2, bufs=bufs,
                                     dV_dtype=dV_dtype)
            return out, g
    step.last_saved = None
    return step


class Throttle:
    """Keeps at most two steps in flight: before enqueueing step i the host
    waits for step i-2's end event (the GPU still has step i-1 queued, so it
    never idles).  Without it the host runs ahead of the device by many steps
    on the memory-group paths, whose side-stream tensors stay reserved by the
    caching allocator until their streams catch up -- and the pool then grows
    (a device allocation, tens of ms) inside the timed region."""

    def __init__(self, torch):
        self.torch, self.ev = torch, []

    def before(self):
        if len(self.ev) >= 2:
            self.ev.pop(0).synchronize()

    def after(self):
        e = self.torch.cuda.Event()
        e.record()
        self.ev.append(e)


def warm_up(step, n, torch):
    """n untimed steps in the timed loop's pattern (the previous step's
    results alive while the next one runs, at most two steps in flight), so
    the caching allocator's pool is settled before timing; none of them live
    across the timed region (one more live generation made the pool grow --
    a device allocation of up to tens of ms -- inside the timed steps)."""
    thr = Throttle(torch)
    out = g = None
    for _ in range(n):
        thr.before()
        out, g = step()
        thr.after()
    del out, g
    torch.cuda.synchronize()


def time_steps(step, steps, world, torch, dev):
    """Device time of `steps` steps on the launch stream (barrier + sync on
    both sides, max over ranks)."""
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
    import gc
    barrier()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()         # no collector pause between launches inside the timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    diag = os.environ.get("BENCH_STEP_TIMES") == "1"
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)] if diag else None
    if diag:
        m0 = torch.cuda.memory_stats()
    h0 = time.perf_counter()
    thr = Throttle(torch)
    # pre-roll (outside the timed region): ~1 ms of GPU spin so that the
    # first timed step's kernels are already queued when e0 fires -- otherwise
    # step 1 also times the host's launch latency on an idle GPU
    torch.cuda._sleep(2_000_000)
    e0.record(stream)
    for i in range(steps):
        thr.before()
        if diag:
            ev[i].record(stream)
        out, g = step()
        thr.after()
    if diag:
        ev[steps].record(stream)
    e1.record(stream)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    gc.enable()
    if diag:
        m1 = torch.cuda.memory_stats()
        keys = ("segment.all.allocated", "num_alloc_retries", "num_device_alloc", "num_device_free")
        print("step ms:", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(steps)],
              f"host enqueue {1e3 * (h1 - h0) / steps:.3f} ms/step",
              {k: m1.get(k, 0) - m0.get(k, 0) for k in keys}, file=sys.stderr)
    barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        m = torch.tensor([ms], device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
    return ms, out, g


def run_ours(args, cfg, world, rank, local):
    import torch
    from paper_2412_09764_b200 import ops
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    per_rank = args.per_rank if world == 1 else 0
    G = world if world > 1 else max(1, per_rank)
    group_path = world > 1 or args.force_group or per_rank > 1
    if "T_global" in cfg and G == 1:
        raise SystemExit(f"{cfg['name']} does not fit one B200 ({cfg['desc']}): run it with "
                         f"--gpus 8 or measure one rank's work with --per-rank 8")
    comm = None
    if world > 1 or args.force_group:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        from paper_2412_09764_b200.group import nccl_group
        comm = CGroup(nccl_group(dist.group.WORLD))
        if args.p2p:
            comm.grp.set_p2p(True)
    t = make_inputs(cfg, dev, G, rank if world > 1 else 0, ops, torch, group_path)
    if per_rank > 1:
        # one rank's work through the library's own group path (C ABI), the
        # collectives replaced by local copies (ml_group_init_loopback)
        comm = CGroup(loopback_group(G, 0, group_others(cfg, G, 0, t, ops, torch), ops, torch))
        if args.p2p:
            comm.grp.set_p2p(True)
    step = build_step(args, cfg, t, ops, torch, comm)
    T_loc = tokens_per_rank(cfg, G)

    clk = ClockSampler(local)          # NVML initialised and queried before the warm-up
    # the memory-group paths allocate per step on several streams: more
    # warm-up steps until the caching allocator's pool is settled
    n_warm = args.warmup if comm is None else max(args.warmup, 8)
    warm_up(step, n_warm, torch)

    # ---- headline: device events around K steps, library timing OFF
    launches0 = ops.launch_count()
    with clk:
        ms, out, g = time_steps(step, args.steps, world, torch, dev)
    launches = ops.launch_count() - launches0
    U = int((g["U"] if isinstance(g, dict) else g.U).item())
    ms_step = ms / args.steps
    # per_rank emulates ONE rank: the group would process G times its tokens
    tokens_per_step = T_loc * (world if world > 1 else 1)

    # ---- per-kernel pass (separate, not timed into the headline): every
    # kernel on the caller's stream so each timing event brackets one launch
    kern_steps = max(1, min(args.steps, 5))
    ops.set_serial(True)
    ops.timing_reset()
    ops.timing_enable(True)
    for _ in range(kern_steps):
        step()
    torch.cuda.synchronize()
    ops.timing_enable(False)
    ops.set_serial(False)
    kern = ops.timing_report()
    coll = coll_report(kern, kern_steps, cfg, G, T_loc, args.mode) \
        if (isinstance(comm, CGroup) and world > 1) else None

    # ---- variant: the compact value gradient stored as bf16 (memlayer.h
    # grad_dtype; fp32 sums rounded once) -- same step otherwise
    variants = None
    if args.dv_dtype == "f32" and cfg["dtype"] == "bf16" and not args.no_variants:
        import copy
        a2 = copy.copy(args)
        a2.dv_dtype = "bf16"
        vstep = build_step(a2, cfg, t, ops, torch, comm)
        warm_up(vstep, n_warm, torch)
        ms_v, _, _ = time_steps(vstep, args.steps, world, torch, dev)
        variants = {"dV_bf16": {"ms_per_step": round(ms_v / args.steps, 4),
                                "value": tokens_per_step / (ms_v / args.steps / 1e3),
                                "note": "compact value gradient stored as bf16 (grad_dtype=ML_BF16; "
                                        "fp32 sums rounded once); the headline keeps fp32 dV"}}
        del vstep

    # ---- t_ref(G): the same rank's work with the collectives removed
    eff = None
    if world > 1:
        saved = step.last_saved
        idx_all, w_all = saved["idx_all"].clone(), saved["w_all"].clone()
        P_loc = idx_all[0].numel() * (idx_all.shape[0] // world)
        lists = torch.empty((world, 2, P_loc), dtype=torch.int32, device=dev)
        for g in range(world):   # every rank's sorted share of the inverse map
            ops.group_sort_local(cfg["S"] ** 2, idx_all.view(world, -1)[g].view(-1, idx_all[0].numel()), g,
                                 out=lists[g])
        others = {"idx_all": idx_all, "w_all": w_all, "lists": lists}
        # t_ref(G): the same rank's work through the same library group path
        # with the collectives replaced by local copies
        lb = loopback_group(world, rank, others, ops, torch)
        if args.p2p:
            lb.set_p2p(True)
        ref_step = build_step(args, cfg, t, ops, torch, CGroup(lb))
        warm_up(ref_step, max(args.warmup, 8), torch)
        ms_ref, _, _ = time_steps(ref_step, args.steps, world, torch, dev)
        eff = {"t_G_ms": round(ms_step, 4), "t_ref_ms": round(ms_ref / args.steps, 4),
               "E": round((ms_ref / args.steps) / ms_step, 4),
               "definition": "SURVEY §8(e): E(G) = t_ref(G) / t_G, t_ref = this rank's work with "
                             "the collectives replaced by local copies (max over ranks)"}

    # ---- e2e: host (pinned) inputs -> device, step, result -> host
    e2e = run_e2e(args, t, step, torch, tokens_per_step, world)
    return dict(value=tokens_per_step / (ms_step / 1e3), ms_step=ms_step, kern=kern,
                kern_steps=kern_steps, launches=launches, clocks=clk.summary(), U=U, e2e=e2e,
                tokens_per_step=tokens_per_step, G=G, T_loc=T_loc, coll=coll, eff=eff,
                variants=variants)


def pin_to_gpu_numa_node(index):
    """Run this process on the CPUs local to the GPU (its PCI device's
    local_cpulist) so the pinned staging buffers allocated next are first
    touched -- and placed -- on the GPU's NUMA node.  Best effort."""
    try:
        import pynvml
        pynvml.nvmlInit()
        bus = pynvml.nvmlDeviceGetPciInfo(pynvml.nvmlDeviceGetHandleByIndex(index)).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        bus = bus.lower()
        if bus.count(":") == 2 and len(bus.split(":")[0]) == 8:   # 00000000:1b:00.0
            bus = bus[4:]
        txt = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        cpus = set()
        for part in txt.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


def run_e2e(args, t, step, torch, tokens_per_step, world):
    """End to end through the public API with HOST buffers: every step copies
    its inputs (q, x, dout) from pinned host memory and copies the result
    `out` back.  The copies run on a copy stream, double-buffered, so step
    i+1's upload overlaps step i's compute (the intended way to feed the
    layer); all of it is inside the timed region."""
    stream = torch.cuda.current_stream()
    names = ("q", "x", "dout")
    aff = os.sched_getaffinity(0)
    numa_cpus = pin_to_gpu_numa_node(t["q"].device.index)
    hostbufs = {n: t[n].cpu().pin_memory() for n in names}
    os.sched_setaffinity(0, aff)           # the pages stay where they were first touched
    h2d = sum(hostbufs[n].numel() * hostbufs[n].element_size() for n in names)
    dbuf = [{n: torch.empty_like(t[n]) for n in names} for _ in range(2)]
    copy = torch.cuda.Stream()      # uploads
    down = torch.cuda.Stream()      # result downloads (separate: a queued download must not
                                    # hold back the next upload)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    # the pinned result buffer is allocated before the timed region (page
    # locking is a synchronous host call, not part of a step)
    out_probe, _ = step({**t, **dbuf[0]})
    out_host = torch.empty(out_probe.shape, dtype=out_probe.dtype, pin_memory=True)
    del out_probe

    def loop(n):
        for e in ev_done:
            e.record(stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        copy.wait_event(e0)
        for i in range(n):
            b = i % 2
            with torch.cuda.stream(copy):
                copy.wait_event(ev_done[b])             # buffer b no longer read by step i-2
                for nm in names:
                    dbuf[b][nm].copy_(hostbufs[nm], non_blocking=True)
                ev_in[b].record(copy)
            stream.wait_event(ev_in[b])
            out, g = step({**t, **dbuf[b]})
            ev_done[b].record(stream)
            with torch.cuda.stream(down):
                down.wait_event(ev_done[b])
                out.record_stream(down)
                out_host.copy_(out, non_blocking=True)
        ev_last = torch.cuda.Event()
        ev_last.record(down)
        stream.wait_event(ev_last)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    loop(3)                          # warm-up of the pipelined loop (first-touch of pinned pages)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ms = loop(max(3, args.steps))   # the first upload (pipeline fill) is inside the timed region
    if world > 1:
        import torch.distributed as dist
        m = torch.tensor([ms], device=t["q"].device)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        ms = float(m.item())
    d2h = out_host.numel() * out_host.element_size()
    return {"value": tokens_per_step / (ms / 1e3), "unit": "tok/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "note": "pinned host inputs uploaded on a copy stream, double-buffered against compute; "
                    "results downloaded on a second copy stream; host buffers on the GPU's NUMA "
                    f"node ({numa_cpus} local CPUs)" if numa_cpus else
                    "pinned host inputs uploaded on a copy stream, double-buffered against compute; "
                    "results downloaded on a second copy stream"}


# ------------------------------------------------- roofline accounting
def bag_bytes(cfg, G, T_loc, U=None):
    """Bytes per launch of the two bag kernels for the per-rank launch at
    group size G (the bag runs over all G*T_loc group tokens on a dv/G
    column slice).  Returns dict with:
      fwd            a5 (+ a6 epilogue at G = 1): rows + (idx, w) + gate/out/y
      bwd_l2_incl    a9, SURVEY §8(d) per-position count: B dy-row gathers per
                     token (served from L2 by design) + V and fp32 dV once
                     per distinct row + metadata + dy
      bwd_hbm        a9 compulsory HBM bytes: V once per distinct row, fp32
                     dV written once, dy read once, sorted key/pos + w (12 B
                     per position), dw partials (16 B per position and slice)
    """
    e = 2 if cfg["dtype"] == "bf16" else 4
    B = cfg["H"] * cfg["k"]
    T_all = T_loc * G
    dvs = cfg["dv"] // G
    P = T_all * B
    fwd = P * (dvs * e + 8) + T_all * dvs * e * (3 if G == 1 else 1)
    u = (U / P) if U else 1.0
    ns = max(1, (dvs * e // 16) // 256)
    bwd_l2 = P * dvs * e + u * P * dvs * (e + 4) + P * (12 + 4 * ns) + T_all * dvs * e
    bwd_hbm = u * P * dvs * (e + 4) + T_all * dvs * e + 12 * P + 16 * ns * P
    return {"fwd": fwd, "bwd_l2_incl": bwd_l2, "bwd_hbm": bwd_hbm, "P": P}


def roofline(res, cfg, peaks):
    kern = res["kern"]
    ks = res["kern_steps"]
    mine = {n: v for n, v in kern.items() if n not in ("cublasLt_gemm", "memset")}
    dom = max(mine, key=lambda n: mine[n][1]) if mine else None
    bb = bag_bytes(cfg, res["G"], res["T_loc"], res["U"])
    hbm = peaks.get("hbm_gbs", 6650.0)
    per = {}
    for n, algo, l2 in (("embbag_fwd_gate", bb["fwd"], None), ("embbag_fwd", bb["fwd"], None),
                        ("embbag_bwd_segreduce", bb["bwd_hbm"], bb["bwd_l2_incl"])):
        if n in kern:
            cnt, tot = kern[n]
            avg_s = tot / cnt / 1e3
            gbs = algo / avg_s / 1e9
            per[n] = {"achieved_GBs": round(gbs, 1), "frac": round(gbs / hbm, 4),
                      "avg_ms": round(tot / cnt, 4), "bytes_per_launch": int(algo)}
            if l2:
                per[n]["l2_inclusive"] = {"bytes_per_launch": int(l2),
                                          "GBs": round(l2 / avg_s / 1e9, 1)}
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if dom and os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(cfg.get("name", ""), {}).get(dom)
        except Exception:
            traffic = None
    if dom in per:
        r = {"bound": "hbm", "kernel": dom, "achieved": per[dom]["achieved_GBs"], "peak": hbm,
             "unit": "GB/s", "frac": per[dom]["frac"], "traffic": traffic,
             "avg_ms": per[dom]["avg_ms"], "bytes_per_launch": per[dom]["bytes_per_launch"],
             "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in peaks
             else "fallback 6650 (B200_PROFILING.md)",
             "timing": f"per-launch CUDA events on the launch stream, separate pass of {ks} steps "
                       "with every kernel on one stream (ml_set_serial)"}
        if "l2_inclusive" in per[dom]:
            r["achieved_note"] = ("bytes that must cross HBM (V once per distinct row, fp32 dV, "
                                  "dy once, 12 B/position metadata, dw partials); l2_inclusive adds "
                                  "the B dy-row gathers per token the kernel serves from L2")
            r["l2_inclusive"] = per[dom]["l2_inclusive"]
        if traffic:
            g = traffic / (per[dom]["avg_ms"] / 1e3) / 1e9
            r["dram"] = {"achieved": round(g, 1), "frac": round(g / hbm, 4), "unit": "GB/s",
                         "source": "ncu dram__bytes (profiles/traffic.json) over the live launch time"}
    else:
        cnt, tot = kern[dom] if dom else (1, 0.0)
        r = {"bound": "alu", "kernel": dom, "achieved": None, "peak": None, "unit": None,
             "frac": None, "traffic": traffic, "avg_ms": tot / max(cnt, 1)}
    # the scoring contraction (a1): tensor-bound
    sc = None
    for n in ("pkm_scores_tc", "pkm_scores_topk_tc"):
        if n in kern:
            cnt, tot = kern[n]
            flops = 2.0 * res["T_loc"] * cfg["H"] * cfg["S"] * cfg["Dk"]
            tf_s = flops / (tot / cnt / 1e3) / 1e12
            pk = peaks.get("bf16_tflops", 1590.0)
            sc = {"kernel": n, "bound": "tensor", "achieved": round(tf_s, 1), "unit": "TFLOP/s",
                  "peak": pk, "frac": round(tf_s / pk, 4), "avg_ms": round(tot / cnt, 4),
                  "flops_per_launch": flops,
                  "peak_source": "MEASURED_PEAKS.json bf16_tflops (cuBLAS, burst)"}
            try:
                util = json.load(open(os.path.join(ROOT, "profiles", "tensor_util.json")))
                sc["tensor_pipe_util_ncu"] = util.get(cfg.get("name", ""), {}).get(n)
            except Exception:
                pass
    return r, per, sc


# ------------------------------------------------------------- oracle arm
def oracle_sample(cfg, T_o, seed=SEED, chunk=256, t0=0):
    """Times the CPU oracle (oracle/) on T_o tokens of the workload (tokens
    t0.., in chunks of `chunk`): full-size tables, value rows and inputs
    regenerated on demand OUTSIDE the timed parts.  Returns (seconds, tokens)."""
    import numpy as np
    from oracle import bag as obag, gate as ogate, pkm as opkm
    from synthetic import gen
    S, dv, D, Dk, H, k = (cfg[n] for n in ("S", "dv", "D", "Dk", "H", "k"))
    dt = cfg["dtype"]
    f64 = lambda a: a.astype(np.float64)
    K1 = f64(gen.tensor(seed, "K1", (H, S, Dk // 2), scale=gen.scale_for("K1", Dk=Dk), dtype=dt))
    K2 = f64(gen.tensor(seed, "K2", (H, S, Dk // 2), scale=gen.scale_for("K2", Dk=Dk), dtype=dt))
    W1 = f64(gen.tensor(seed, "W1", (D, dv), scale=gen.scale_for("W1", D=D), dtype=dt))
    W2 = f64(gen.tensor(seed, "W2", (dv, D), scale=gen.scale_for("W2", dv=dv), dtype=dt))
    el, done = 0.0, 0
    while done < T_o:
        n = min(chunk, T_o - done)
        toks = np.arange(t0 + done, t0 + done + n)
        rows = (toks[:, None] * H + np.arange(H)[None, :]).reshape(-1)
        q = f64(gen.rows(seed, "q", rows, Dk, dtype=dt)).reshape(n, H, Dk)
        x = f64(gen.rows(seed, "x", toks, D, dtype=dt))
        dout = f64(gen.rows(seed, "dout", toks, D, dtype=dt))
        t_0 = time.perf_counter()
        idx, score, w = opkm.pkm_lookup(q, K1, K2, k)
        el += time.perf_counter() - t_0
        bidx = idx.reshape(n, H * k)
        bw = w.reshape(n, H * k)
        uniq, lidx = np.unique(bidx, return_inverse=True)
        Vrows = f64(gen.rows(seed, "V", uniq, dv, dtype=dt))      # untimed: input synthesis
        lidx = lidx.reshape(n, H * k)
        t_0 = time.perf_counter()
        y = obag.embbag_fwd(Vrows, lidx, bw)
        out, g, z = ogate.gate_fwd(x, y, W1, W2)
        gb = ogate.gate_bwd(dout, x, y, g, W1, W2)
        rows_, dV, dw = obag.embbag_bwd(Vrows, lidx, bw, gb["dy"])
        dq, dK1, dK2, _ = opkm.pkm_bwd(q, K1, K2, idx, w, dw.reshape(n, H, k))
        el += time.perf_counter() - t_0
        done += n
    return el, T_o


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def timed_oracle(cfg, T_o, threads):
    """The oracle on T_o tokens with the BLAS pool limited to `threads` (the
    oracle's only parallel part: numpy fp64 matmuls)."""
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=threads):
            return oracle_sample(cfg, T_o)
    except ImportError:
        return oracle_sample(cfg, T_o)


def cpu_baseline(cfg, T_o):
    n = host_threads()
    el_n, tok = timed_oracle(cfg, T_o, n)
    el_1, tok1 = timed_oracle(cfg, max(1, T_o // 2), 1)
    return {"value": tok / el_n, "unit": "tok/s", "cores": n, "kind": "oracle",
            "sample": f"{tok} tokens (chunks of 256) of {cfg['desc']}: full-size tables, rows "
                      f"regenerated on demand outside the timed parts; numpy fp64, BLAS pool of "
                      f"{n} threads (the matmuls are the oracle's only parallel part)",
            "seconds": round(el_n, 3), "cpu_model": cpu_model(),
            "single_thread": {"value": tok1 / el_1, "unit": "tok/s", "cores": 1,
                              "tokens": tok1, "seconds": round(el_1, 3)}}


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return None
    T_o = args.ref_tokens
    n = host_threads()
    for _ in range(args.warmup):
        timed_oracle(cfg, max(2, T_o // 4), n)
    tot, toks = 0.0, 0
    for _ in range(args.steps):
        el, m = timed_oracle(cfg, T_o, n)
        tot += el
        toks += m
    v = toks / tot
    return {"metric": METRIC, "value": v, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": dict(config_keys(cfg, cfg.get("name", "c2"), 1, "single GPU",
                                       tokens_per_rank(cfg, 1) if "T" in cfg else cfg["T_global"]),
                           tokens_per_step_sample=T_o),
            "cpu_baseline": {"value": v, "unit": "tok/s", "kind": "oracle", "cores": n,
                             "cpu_model": cpu_model(),
                             "sample": f"{T_o} tokens per step of {cfg['desc']}"},
            "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------- main
def config_keys(cfg, cfg_name, G, parallelism, T_loc):
    """The workload description shared by both arms' JSON lines."""
    return {"workload": cfg["desc"], "config": cfg_name, "tokens_per_rank": T_loc,
            "global_tokens": T_loc * G, "N_values": cfg["S"] ** 2, "value_dim": cfg["dv"],
            "heads": cfg["H"], "k": cfg["k"], "key_dim": cfg["Dk"], "gated": True,
            "parallelism": parallelism,
            "l2": "inputs_larger_than_L2 (value table >= 4 GiB vs 126 MB L2; no flush)",
            "seed": SEED}


def dry_run(args, world, rank):
    """CPU rendezvous check of the multi-rank launch (gloo): every rank joins,
    barriers, and reduces a per-rank number with MAX; rank 0 prints."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "world_size": dist.get_world_size(),
                          "max_over_ranks": float(t.item())}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--mode", default="alltoall", choices=["alltoall", "allgather"])
    ap.add_argument("--p2p", action="store_true",
                    help="N > 1, mode alltoall: the fused peer-memory forward exchange "
                         "(ml_group_set_p2p: bag kernels store into the owners' regions) instead "
                         "of NCCL point-to-point steps")
    ap.add_argument("--per-rank", type=int, default=0,
                    help="on one GPU: time one rank's work of a G-rank group (collectives removed)")
    ap.add_argument("--cpu-tokens", type=int, default=1024)
    ap.add_argument("--ref-tokens", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--qk-norm", action="store_true", help="qk-normalisation (SURVEY f2)")
    ap.add_argument("--no-state", action="store_true",
                    help="backward sorts the indices itself (no forward-built state)")
    ap.add_argument("--dv-dtype", default="f32", choices=["f32", "bf16"],
                    help="storage of the compact value gradient (memlayer.h grad_dtype)")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the bf16-dV variant timing")
    ap.add_argument("--force-group", action="store_true",
                    help="run the memory-group (NCCL) path even at N=1 (torchrun)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU: only the multi-rank launch + rendezvous (gloo), no GPU work")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(respawn_under_torchrun(args.gpus))
    world, rank, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch with matching "
              f"--nproc-per-node", file=sys.stderr)
        sys.exit(2)
    if args.dry_run:
        dry_run(args, world, rank)
        return
    if args.warmup < 3:
        args.warmup = 3
    cfg_name = args.config or "c2"
    cfg = dict(CONFIGS[cfg_name], name=cfg_name)

    if args.impl == "reference":
        line = run_reference(args, cfg, world, rank)
        if line:
            print(json.dumps(line), flush=True)
        return

    res = run_ours(args, cfg, world, rank, local)
    if rank != 0:
        return
    peaks = load_peaks()
    G = res["G"]
    roof, per, scoring = roofline(res, cfg, peaks)
    cb = None
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(cfg, args.cpu_tokens if cfg_name != "c1" else cfg["T"])
    bb = bag_bytes(cfg, G, res["T_loc"], res["U"])
    if world > 1:
        par = f"memory-group dim-shard G={G} ({args.mode}), NCCL" + (
            " + fused peer-memory forward exchange" if args.p2p and args.mode == "alltoall" else "")
    elif args.per_rank > 1:
        par = (f"one rank of a G={G} memory group on one GPU (collectives replaced by local "
               f"copies: SURVEY §8(e) t_ref(G)), {args.mode}" +
               (", fused peer-store exchange" if args.p2p and args.mode == "alltoall" else ""))
    elif args.force_group:
        par = f"memory-group path G=1 ({args.mode}), NCCL"
    else:
        par = "single GPU"
    line = {
        "metric": METRIC, "value": res["value"], "unit": "tok/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_step"],
        "higher_is_better": True, "scaling": "strong" if "T_global" in cfg else "weak",
        "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
        "config": dict(config_keys(cfg, cfg_name, world if world > 1 else 1, par, res["T_loc"]),
                       qk_norm=bool(args.qk_norm), per_rank_G=args.per_rank or None,
                       dV_dtype=args.dv_dtype,
                       unique_rows_per_position=round(res["U"] / bb["P"], 4)),
        "roofline": roof,
        "scoring_roofline": scoring,
        "bag_kernels": per,
        "kernel_ms_per_step": {n: round(v[1] / res["kern_steps"], 4) for n, v in sorted(
            res["kern"].items(), key=lambda kv: -kv[1][1])},
        "kernel_timing": "separate pass, kernels serialised on the caller's stream (ml_set_serial)",
        "per_rank": ({"G": G, "t_ref_ms": round(res["ms_step"], 4),
                      "group_tokens_per_step": G * res["T_loc"],
                      "group_tok_s_at_E1": G * res["T_loc"] / (res["ms_step"] / 1e3),
                      "note": "value = this one rank's tokens per second"}
                     if (world == 1 and args.per_rank > 1) else None),
        "variants": res["variants"],
        "collectives": res["coll"],
        "scaling_efficiency": res["eff"],
        "cpu_baseline": cb,
        "e2e": res["e2e"],
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "paper_context": "PAPER.md P:176: custom EmbeddingBag fwd 3 TB/s on H100 (3.35 TB/s spec)",
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
