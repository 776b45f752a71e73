"""EM-step throughput of the SVHN-shaped Poon-Domingos EiNet (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one EM update (forward + responsibility back-pass over the rank's
batch shard, one NCCL all-reduce of the packed fp64 statistics when N > 1,
fused M-step) -- the reference ``trainer.em_stochastic_step``
(trainer.py:99-117) on the GPU. The K timed steps run through the public
``trainer.em_stochastic_steps`` on the HBM-resident batch: every step is a
complete update whose mean LL and error words are logged on the device and
read back once after the K steps (no host round trip between steps). Workload: config C3 of BASELINE.json
(32x32x3 lifted PD, delta 8 vertical, K=40, Gaussian image-mode leaves),
synthetic image data, a fixed per-GPU batch (weak scaling). Inputs are larger
than L2 (16384 x 3072 fp32 = 201 MB > 126 MB), so no flush is needed.

``e2e`` runs the same steps through the public ``trainer.em_stochastic_steps``
from pinned host memory: the batch ships as the u8 pixels it was quantised
from (x = k/255, the reference's EIND1 u8 dataset payload, modelio.py:145-166)
and is decoded on the device (``einet_decode_u8``, bit-identical values);
``e2e.fp32_host_input`` is the same leg fed the fp32 host array.

``--impl reference`` times the CPU restatement of the reference's EM step
(oracle/einet_oracle.py; the Python reference itself cannot travel to the GPU
box) on all host cores with a bounded sample per step.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EM-step samples/s, SVHN-shape PD EiNet K=40"
UNIT = "samples/s"
CONFIG = "C3"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=16384, help="samples per GPU per step")
    ap.add_argument("--chunk", type=int, default=16384)
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--small-batch", type=int, default=1,
                    help="also time the 4096-sample batch of SURVEY.md 8d (secondary field)")
    ap.add_argument("--cpu-sample", type=int, default=96,
                    help="samples per oracle EM step for the CPU legs")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms during a region (NVML;
    nvidia-smi as the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reason bits)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            n = self._nvml
            sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
            mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
            bits = n.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return float(sm), float(mx), int(bits)
        out = subprocess.run(
            ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
             "clocks_event_reasons.active", "--format=csv,noheader,nounits"],
            capture_output=True, text=True, timeout=5).stdout.strip()
        sm, mx, bits = [v.strip() for v in out.split(",")]
        return float(sm), float(mx), int(bits, 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.rows.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        # the timed loop holds the GIL between launches: a short switch
        # interval lets the sampling thread in every millisecond
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(0.001)
        try:
            self.rows.append(self._sample())
        except Exception:
            pass
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        sys.setswitchinterval(self._switch)
        try:
            self.rows.append(self._sample())
        except Exception:
            pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({n for _, _, bits in self.rows for n, m in self.REASONS.items()
                          if bits & m})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# ---------------------------------------------------------------------------
# algorithmic work per sample, per kernel class
# ---------------------------------------------------------------------------

def work_per_sample(circuit):
    """Algorithmic flops and HBM bytes per sample for each kernel class
    (SURVEY.md 8d)."""
    k = circuit.k
    d, r = circuit.d_vars, circuit.num_replicas
    ein = 0
    for layer in circuit.layers[1:]:
        if type(layer).__name__ == "EinsumLayer":
            ein += len(layer.left_src) * layer.k_out * k * k
    leaf_elems = d * k * r
    return {
        # (x - mu)^2 / (2 var): 2 FMA per (var, k); x read once
        "leaf_fwd": {"flops": 4 * leaf_elems, "bytes": 4 * d, "tc": False},
        "einsum_fwd": {"flops": 2 * ein, "bytes": 0, "tc": True},
        "einsum_wstats": {"flops": 2 * ein, "bytes": 0, "tc": True},
        "einsum_childrho": {"flops": 4 * ein, "bytes": 0, "tc": True},
        # rho*y and rho*y^2 per (var, k); x read once
        "leaf_stats": {"flops": 4 * leaf_elems, "bytes": 4 * d, "tc": False},
    }


def load_peaks():
    """(peaks dict, source): MEASURED_PEAKS.json (driver-written), else the
    profiling recipe's stated fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            doc = json.load(f)
        return {"hbm_gbs": doc.get("hbm_gbs", 6650.0), "bf16_tflops": doc.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": doc.get("bf16_tflops_sustained", 1400.0),
                "sm_max_mhz": doc.get("sm_max_mhz", 1965.0)}, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


# ncu DRAM traffic (read + write bytes per launch) of the dominant kernels,
# from the committed --set full capture
# (name prefixes; scripts/kernel_traffic.py writes the file from an ncu launch list)
KERNEL_TRAFFIC = {"leaf_fwd": "k_leaf_fwd_i8", "leaf_stats": "k_leaf_stats_tc",
                  "einsum_wstats": "k_wstats_tc", "einsum_childrho": "k_contract_tc",
                  "einsum_fwd": "k_contract_tc"}


def kernel_traffic(name):
    path = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    try:
        with open(path) as f:
            doc = json.load(f)
        v = [b for k, e in doc.items() if k.startswith(KERNEL_TRAFFIC[name])
             for b in e["dram_bytes_per_launch"]]
        return max(v) if v else None
    except Exception:
        return None


def class_fractions(name, w, B, per_step_ms, groups, peaks):
    """Roofline fractions of one kernel class from its device time: HBM
    (algorithmic bytes) and tensor (algorithmic flops, and the 3 MMAs a
    3xBF16 product issues) against the measured peaks."""
    out = {}
    t = per_step_ms / 1e3
    if w["bytes"]:
        gbs = w["bytes"] * B / t / 1e9
        out["hbm_gbs"] = gbs
        out["hbm_frac"] = gbs / peaks["hbm_gbs"]
    if w.get("tc"):
        tf = w["flops"] * B / t / 1e12
        out["tflops"] = tf
        out["tc_frac"] = tf / peaks["bf16_tflops"]
        out["tc_frac_issued_3xbf16"] = 3 * tf / peaks["bf16_tflops"]
    return out


def step_roofline(circuit, B, ms_step, peaks):
    """Whole-step roofline of SURVEY.md 8d: t_roof = max(F_TC / P_TC,
    F_CC / P_FP32, bytes / BW) per sample, fraction = t_roof / t_measured.
    `survey` counts the leaf work on CUDA cores (the survey's formula, FP32
    SIMT peak provisional: 148 SM x 128 lanes x 2 x max clock); `as_built`
    counts it on tensor cores, as this build runs it (INT8 leaf forward,
    3xTF32 leaf statistics), against the bf16 peak (conservative)."""
    k, d, r = circuit.k, circuit.d_vars, circuit.num_replicas
    ein = sum(len(l.left_src) * l.k_out * k * k for l in circuit.layers[1:]
              if type(l).__name__ == "EinsumLayer")
    f_tc = 3 * 2 * ein                     # forward + W statistics + child responsibilities
    f_leaf = 4 * d * k * r + 4 * d * k * r  # leaf forward + leaf statistics
    f_rest = 4 * ein // max(k, 1)          # exp / log / outer-product glue (small)
    bytes_ = 4 * d                         # x read once
    p_tc = peaks["bf16_tflops"] * 1e12
    p_cc = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6
    bw = peaks["hbm_gbs"] * 1e9
    t_meas = ms_step / 1e3 / B
    res = {}
    for name, tc, cc in (("survey", f_tc, f_leaf + f_rest), ("as_built", f_tc + f_leaf, f_rest)):
        comps = {"tensor_s": tc / p_tc, "cuda_core_s": cc / p_cc, "hbm_s": bytes_ / bw}
        t_roof = max(comps.values())
        res[name] = {"t_roof_ns_per_sample": t_roof * 1e9,
                     "bound": max(comps, key=comps.get).replace("_s", ""),
                     "ceiling_samples_per_s": 1.0 / t_roof, "frac": t_roof / t_meas}
    res["t_measured_ns_per_sample"] = t_meas * 1e9
    res["fp32_simt_peak"] = "provisional (not in MEASURED_PEAKS.json)"
    return res


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference EM step)
# ---------------------------------------------------------------------------

def _oracle_setup(config, n, seed):
    from paper_2004_06231_b200 import engine
    from paper_2004_06231_b200.compiler import compile_graph
    from paper_2004_06231_b200.data import config as cfg
    from oracle import einet_oracle as O
    rg, fam, k, gen = cfg(config)
    circuit = compile_graph(rg, k)
    x = gen(n, seed=seed).astype(np.float32).astype(np.float64)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=x)
    return circuit, fam.to_dict(), x, O.OracleParams(ein, mix, phi)


_WORKER = {}


def _oracle_worker_init(config, n, seed):
    _WORKER["model"] = _oracle_setup(config, n, seed)


def _oracle_shard(args):
    """E-step of one shard with the current parameters (engine.py:143-328)."""
    params, lo, hi = args
    from oracle import einet_oracle as O
    circuit, fam, x, _ = _WORKER["model"]
    tr = O.forward(circuit, params, fam, x[lo:hi])
    return O.backward(circuit, params, fam, tr)


def cpu_reference_steps(config, n, steps, warmup, procs):
    """Reference EM step (trainer.py:99-117) restated in oracle/, sharded over
    `procs` worker processes that keep the model resident; the parent merges
    the statistics (a sum, engine.py:228-236) and applies the M-step."""
    import multiprocessing as mp
    from oracle import einet_oracle as O
    circuit, fam, x, p = _oracle_setup(config, n, 0)
    bounds = np.linspace(0, n, procs + 1).astype(int)
    spans = [(int(bounds[i]), int(bounds[i + 1])) for i in range(procs)
             if bounds[i + 1] > bounds[i]]
    times = []
    ctx = mp.get_context("fork")
    with ctx.Pool(len(spans), initializer=_oracle_worker_init, initargs=(config, n, 0)) as pool:
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            parts = pool.map(_oracle_shard, [(p, lo, hi) for lo, hi in spans])
            st = parts[0]
            for q in parts[1:]:
                st.merge(q)
            p = O.apply_update(circuit, p, fam, st, 0.5)
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
    return times


def cpu_baseline(config, n):
    """Single-core oracle EM step on a bounded sample (~10-30 s of CPU work)."""
    from oracle import einet_oracle as O
    circuit, fam, x, p = _oracle_setup(config, n, 0)
    t0 = time.perf_counter()
    O.em_step(circuit, p, fam, x, 0.5)
    first = time.perf_counter() - t0
    reps = max(1, min(5, int(15.0 / max(first, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(reps):
        O.em_step(circuit, p, fam, x, 0.5)
    dt = (time.perf_counter() - t0) / reps
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{reps}+1 oracle EM steps of {n} {config} samples (numpy fp64, "
                      f"oracle/einet_oracle.py), {dt:.2f} s per step"}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = max(1, len(os.sched_getaffinity(0)))
    n = max(procs * 32, args.cpu_sample)
    steps, warmup = max(1, min(args.steps, 3)), min(args.warmup, 1)
    times = cpu_reference_steps(args.config, n, steps, warmup, procs)
    sec = statistics.median(times)
    value = n / sec
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(times), "warmup": warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} SVHN-shape 32x32x3 PD EiNet K=40, "
                                   f"delta 8 vertical, Gaussian leaves, EM lambda 0.5",
                       "batch_per_step": n, "procs": procs},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": f"{n} samples per EM step, sharded over {procs} "
                                       f"processes (oracle/einet_oracle.py)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2004_06231_b200 import _native, engine, trainer
    from paper_2004_06231_b200.compiler import compile_graph
    from paper_2004_06231_b200.data import config as cfg
    from paper_2004_06231_b200.model import EinetModel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    dev = torch.device("cuda", local)

    rg, fam, k, gen = cfg(args.config)
    circuit = compile_graph(rg, k)
    B = args.batch
    x64 = gen(B, seed=1000 + rank)
    x_host = torch.from_numpy(x64.astype(np.float32)).pin_memory()
    # the same batch as the image bytes it was quantised from (k / 255, an
    # EIND1 u8 payload): the e2e leg ships these and decodes on the device
    x_u8 = torch.from_numpy(np.rint(x64 * 255.0).astype(np.uint8)).pin_memory()
    # the reference caller's type: a float64 NumPy batch (load_dataset returns
    # float64, modelio.py:137-168); packed by einet_pack_f64 inside the
    # public call
    x_np64 = np.ascontiguousarray(x64)
    x_dev = x_host.to(dev)
    init_x = gen(4096, seed=7).astype(np.float32).astype(np.float64)
    ein, mix, phi = engine.init_parameters_host(circuit, fam, seed=0, data=init_x)
    params = engine.Parameters.from_numpy(circuit, fam, ein, mix, phi, device=dev)
    model = EinetModel(circuit, params, fam)

    def step(x):
        return trainer.em_stochastic_step(model, x, 0.5, chunk=args.chunk,
                                          process_group=group)

    for _ in range(args.warmup):
        step(x_dev)
    torch.cuda.synchronize()

    def timed(fn, k):
        if group is not None:
            dist.barrier()
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(k):
            fn()
        stop.record()
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        ms = torch.tensor([start.elapsed_time(stop)], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    # kernels per step: counted on one uncaptured step (the timed steps replay
    # the CUDA graph of this launch sequence plus its last node, the step-log
    # kernel einet_log_step of the pipelined em_stochastic_steps)
    os.environ["EINET_CUDA_GRAPHS"] = "0"
    launches0 = _native.launch_count()
    step(x_dev)
    launches = _native.launch_count() - launches0 + 1
    os.environ.pop("EINET_CUDA_GRAPHS")
    step(x_dev)
    torch.cuda.synchronize()
    # the timed steps: the public pipelined API on the HBM-resident batch (each
    # step a full EM update whose LL and error words are logged on the device;
    # one host read at the end)
    trainer.em_stochastic_steps(model, [x_dev] * 2, 0.5, chunk=args.chunk, process_group=group)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ms = timed(lambda: trainer.em_stochastic_steps(model, [x_dev] * args.steps, 0.5,
                                                        chunk=args.chunk,
                                                        process_group=group), 1)

    # end to end: the pinned host batch goes through the public API each step
    # (host -> device copy inside trainer.em_stochastic_steps, overlapped with
    # the previous step), every step's mean LL read back
    e2e_steps = max(3, args.steps)  # the pipelined API fills once per call

    def e2e_leg(xh):
        # the public multi-step API: batch i+1's host->device copy overlaps step i,
        # no host wait between steps (N > 1: the NCCL all-reduces between graphs)
        return timed(lambda: trainer.em_stochastic_steps(model, [xh] * e2e_steps, 0.5,
                                                          chunk=args.chunk,
                                                          process_group=group), 1)

    # the u8 and fp32 host batches decode to the same device values
    assert torch.equal(engine.as_device_batch(x_u8.to(dev)), x_dev)
    for xh in (x_u8, x_host):  # staging buffers and their graphs exist before timing
        trainer.em_stochastic_steps(model, [xh] * 2, 0.5, chunk=args.chunk, process_group=group)
    ms_e2e = e2e_leg(x_u8)
    ms_e2e_f32 = e2e_leg(x_host)
    # the link the e2e leg crosses: pinned host -> device copy of one step's
    # u8 batch, alone (best of 5), for the e2e leg's bound
    xd_u8 = torch.empty_like(x_u8, device=dev)
    h2d_ms = []
    for _ in range(5):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        xd_u8.copy_(x_u8, non_blocking=True)
        ev1.record()
        torch.cuda.synchronize()
        h2d_ms.append(ev0.elapsed_time(ev1))
    h2d_link_gbs = x_u8.numel() / (min(h2d_ms) / 1e3) / 1e9
    del xd_u8
    f64_steps = 10
    trainer.em_stochastic_steps(model, [x_np64] * 2, 0.5, chunk=args.chunk, process_group=group)
    ms_e2e_f64 = timed(lambda: trainer.em_stochastic_steps(model, [x_np64] * f64_steps, 0.5,
                                                            chunk=args.chunk,
                                                            process_group=group), 1)

    # secondary: the SURVEY.md 8d weak-scaling batch (4096 per GPU) and the
    # paper's batch (500), same model, device-resident
    small = []
    if args.small_batch:
        for sb in (4096, 500):
            if sb >= args.batch:
                continue
            xs = x_dev[:sb]
            sstep = lambda n, xs=xs, sb=sb: trainer.em_stochastic_steps(
                model, [xs] * n, 0.5, chunk=sb, process_group=group)
            sstep(3)
            n_sb = max(args.steps, 20)
            ms_small = timed(lambda: sstep(n_sb), 1)
            small.append({"batch_per_gpu": sb, "chunk": sb, "steps": n_sb,
                          "value": world * sb * n_sb / (ms_small / 1e3),
                          "ms_per_step": ms_small / n_sb})

    # per-kernel-class device time of the same step (CUDA events, separate pass)
    _native.profile_enable(True)
    prof_steps = 3
    for _ in range(prof_steps):
        step(x_dev)
    torch.cuda.synchronize()
    prof = _native.profile_read()
    _native.profile_enable(False)

    if rank != 0:
        if group is not None:
            dist.destroy_process_group()
        return

    value = world * B * args.steps / (ms / 1e3)
    e2e = world * B * e2e_steps / (ms_e2e / 1e3)
    e2e_f32 = world * B * e2e_steps / (ms_e2e_f32 / 1e3)
    e2e_f64 = world * B * f64_steps / (ms_e2e_f64 / 1e3)
    peaks, peak_kind = load_peaks()
    work = work_per_sample(circuit)
    classes = {}
    for name, (tot_ms, cnt) in prof.items():
        per_step = tot_ms / prof_steps
        w = work.get(name)
        c = {"ms_per_step": per_step, "launch_groups_per_step": cnt / prof_steps, "share": None}
        if w is not None:
            c.update(class_fractions(name, w, B, per_step, cnt / prof_steps, peaks))
        classes[name] = c
    total_prof = sum(c["ms_per_step"] for n, c in classes.items() if n not in ("prepare",))
    for c in classes.values():
        c["share"] = c["ms_per_step"] / total_prof if total_prof else None
    # The roofline object reports the dominant kernel: k_contract_tc, the
    # tcgen05 EinsumLayer contraction (north_star), whose launches make up the
    # einsum_fwd and einsum_childrho classes (3 of the 4 GEMM passes of a
    # step: 6 * sum_rows Ko K^2 flops per sample); the largest single class is
    # named beside it.
    largest = max((n for n in classes if n in work), key=lambda n: classes[n]["ms_per_step"])
    ct = [n for n in ("einsum_fwd", "einsum_childrho") if n in prof]
    if ct:
        top = "einsum_contraction (k_contract_tc: einsum_fwd + einsum_childrho)"
        tw = {"flops": sum(work[n]["flops"] for n in ct), "bytes": 0, "tc": True}
        t_step = sum(prof[n][0] for n in ct) / prof_steps
        ct_launches = sum(prof[n][1] for n in ct) / prof_steps
        per_launch_ms = t_step / ct_launches
        groups = ct_launches
        traffic_key = "einsum_fwd"
    else:
        top = largest
        tw = work[top]
        per_launch_ms = prof[top][0] / prof[top][1]
        groups = prof[top][1] / prof_steps
        traffic_key = top
    if tw.get("tc"):
        achieved = tw["flops"] * B / groups / (per_launch_ms / 1e3) / 1e12
        roof = {"kernel": top, "bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["bf16_tflops"],
                "frac_issued_3xbf16": 3 * achieved / peaks["bf16_tflops"],
                "peak_source": f"bf16 dense, {peak_kind}"}
    else:
        achieved = tw["bytes"] * B / groups / (per_launch_ms / 1e3) / 1e9
        roof = {"kernel": top, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "peak_source": f"HBM copy, {peak_kind}"}
    roof["largest_class"] = largest
    roof["traffic"] = kernel_traffic(traffic_key)
    if roof["traffic"] is not None:
        roof["traffic_source"] = "profiles/kernel_traffic.json (ncu dram read+write bytes/launch)"
    roof["algorithmic_bytes"] = tw["bytes"] * B / groups
    roof["per_launch_ms"] = per_launch_ms
    roof["step"] = step_roofline(circuit, B, ms / args.steps, peaks)

    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config, args.cpu_sample)
        except Exception as exc:  # reported, never fatal for the GPU number
            cpu = {"value": None, "error": repr(exc)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "mixed: exact u8 x s8 leaf forward, 3xBF16 contractions (fp32-equivalent), fp64 statistics and M-step",
        "data": "synthetic",
        "config": {"workload": f"{args.config} SVHN-shape 32x32x3 PD EiNet K=40, delta 8 "
                               f"vertical, Gaussian image-mode leaves, EM lambda 0.5",
                   "batch_per_gpu": B, "global_batch": B * world, "chunk": args.chunk,
                   "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2 (B*3072*4 bytes per GPU > 126 MB)"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(B * rg.d_vars),
                "d2h_bytes_per_step": 48, "steps": e2e_steps,
                "h2d_gbs": B * rg.d_vars * e2e / B / 1e9,
                "h2d_link_gbs": h2d_link_gbs,
                "bound": ("pcie h2d (u8 batch copy, overlapped with the device step)"
                          if B * rg.d_vars * e2e / B / 1e9 > 0.85 * h2d_link_gbs else "device"),
                "input": "pinned host u8 pixels (EIND1 payload, x = k/255), copied and "
                         "decoded on the device inside trainer.em_stochastic_steps",
                "fp32_host_input": {"value": e2e_f32,
                                    "h2d_bytes_per_step": int(B * rg.d_vars * 4)},
                "f64_numpy_input": {"value": e2e_f64, "steps": f64_steps,
                                    "h2d_bytes_per_step": int(B * rg.d_vars * 1),
                                    "input": "float64 NumPy batch (the reference caller's "
                                             "type): packed inside the timed call by "
                                             "einet_pack_f64 on all host threads (one byte "
                                             "per value on the u8 grid, as here; else fp32) "
                                             "into pinned halves, batch i+1 packed while "
                                             "step i runs"}},
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernels": classes,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "secondary_batches": small,
    }
    print(json.dumps(line), flush=True)
    if group is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
