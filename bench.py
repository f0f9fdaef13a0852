#!/usr/bin/env python
"""Benchmark of the co-located token step on B200 (driver contract).

Workload (BASELINE.json configs[2], "C3", the largest single-GPU config): eight
co-located Llama-shaped models [1.1B, 3B, 7B, 1.1B, 3B, 7B, 1.1B, 3B]
(random-init weights, synthetic prompts) on one B200, each on its own
execution lane with an SM quota in proportion to its streamed weight bytes,
all drawing on the GPU's VMM KV pool.

  step    one instance step of the co-located schedule (the planned decode of
          that instance's batch of 8, or the prefill of a newly admitted
          request), launched through the mesh_gpu C ABI; every instance keeps up
          to 4 steps queued on its own lane and is re-fed as its steps retire.
          Every admission and completion re-sizes the instance's KV target by
          the reference's rule (m_require + 20 % watermark, memory.cpp:19-36):
          KV grow (VMM map) and shrink (compaction kernel) run inside the timed
          region.
  value   co-located tokens/s over the K timed steps (device-resident inputs),
          counting only tokens of requests whose emissions met the TTFT/TPOT
          SLO on the device timeline (CUDA events, mesh_gpu_timer_mark), max
          over ranks.
  e2e     the same metric through the reference-facing plugin API (llmmesh.h:
          llm_experiment_run with the GPU attached, runtime.clock = "wall") on
          the C3 bursty trace (scenarios/c3_b200: the acceptance overload
          generator's three phases in 30 s) at several load scales: the control
          plane admits, scales KV and cold-starts instances; step completions
          and emission times are CUDA events, so SLO compliance is measured,
          not priced. value = SLO tokens / host wall s, the best over the load
          scales whose compliance is >= 0.99; models/GPU reported.
  roofline  dominant kernel = the persistent decode kernel; algorithmic bytes
          per launch = W_m + sum_i L_i C_m + B C_m + B d_m 2 over the
          timed device span (lanes overlap) and over its own CUDA-event time.

`--impl reference` and `cpu_baseline`: the reference artifact prices token
steps from tables and computes no tokens, so the CPU path that
*executes* the co-located step is the oracle's batched CPU decode
(oracle/cpu_decode.c, all host threads) on the same C3 instance steps: the
same models, batch 8, contexts drawn from the same length set (kind "port");
the reference simulator itself (oracle/_ref) is timed beside it on the C3
trace ("reference_simulator").
Multi-GPU (torchrun): every rank runs an independent co-located node (instances
shard by placement, no collective): weak scaling.
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

C3_DIR = os.path.join(ROOT, "scenarios", "c3_b200")
METRIC = "co-located tokens/s at TTFT/TPOT SLO per B200"
UNIT = "tokens/s"
MODELS = ["1b", "3b", "7b", "1b", "3b", "7b", "1b", "3b"]
BATCH = 8
LANES = int(os.environ.get("MESH_BENCH_LANES", "8"))  # one execution lane per co-located instance
KV_POOL = 100 << 30     # value leg: KV pool per device
# e2e / fleet: the control plane's KV budget (node mem 150 GB - the resident models' weights, ~97 GB)
# plus each instance's physical rounding to whole granules (<= 256 MiB x ~66 instances); 53 GB of
# weights + 116 GB of KV + lane scratch fit the B200's 179 GB
E2E_KV_POOL = 116 << 30
KV_PREALLOC_GB = 96     # e2e: KV arena backed at open (params of the 8 resident models + this fit HBM with scratch)
# e2e: 256 MiB physical KV granules. cuMemMap / cuMemSetAccess cost milliseconds per call once dozens
# of instances hold mappings; at 80 instance starts 32 MiB granules spent 7.8 s of host time in them,
# 128 MiB 4.3 s, 512 MiB 2.4 s (tools/e2e_c3.py, MESH_GPU_KV_GRANULE_MB)
KV_GRANULE_MB = 256
E2E_SCALES = [int(x) for x in os.environ.get("MESH_BENCH_E2E_SCALES", "10,12,14,16").split(",")]
WATERMARK = 20.0
CPU_SAMPLE_S = 15.0     # bounded CPU baseline sample
CPU_MAX_SEQ = 1160      # >= the longest I + O of the length set (1139)


def profiler_region(on: bool) -> None:
    """MESH_PROFILE_REGION=1: cudaProfilerStart/Stop around the timed region, so
    `ncu --profile-from-start off` captures exactly the timed launches."""
    if not os.environ.get("MESH_PROFILE_REGION"):
        return
    import ctypes
    try:  # driver API: acts on the context current on this thread (the data plane's primary context)
        drv = ctypes.CDLL("libcuda.so.1")
    except OSError:
        return
    (drv.cuProfilerStart if on else drv.cuProfilerStop)()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Dist:
    def __init__(self):
        self.ws, self.rank, self.local = dist_env()
        self.pg = None
        if self.ws > 1:
            import torch
            import torch.distributed as dist
            backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.dist, self.torch, self.backend = dist, torch, backend
            # host-side barrier for the fleet leg: an NCCL barrier would leave a kernel spinning
            # on every waiting rank's GPU -- the GPUs rank 0 is driving -- and a persistent decode
            # grid needs all of its quota's SMs co-resident
            self.cpu_pg = dist.new_group(backend="gloo") if backend == "nccl" else None

    def barrier(self, host: bool = False):
        if self.ws > 1:
            self.dist.barrier(group=self.cpu_pg if host else None)

    def reduce(self, x: float, op: str) -> float:
        if self.ws == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device=f"cuda:{self.local}" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.ws > 1:
            self.dist.destroy_process_group()


class Solo:
    """Dist stand-in for work one rank does alone (no collectives)."""
    ws, rank = 1, 0

    def barrier(self, host: bool = False):
        pass

    def reduce(self, x: float, op: str) -> float:
        return x


class Clocks:
    """Clock / throttle-reason sampling DURING the timed region (B200_PROFILING.md
    clocks line). NVML is polled every 10 ms from a thread, and sampled once more
    synchronously at both edges of the region, so even a sub-second region has
    samples; nvidia-smi (100 ms, slow to start) is the fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, {reasons})
        self.proc = None
        self.nv = None
        self.stop = threading.Event()

    def _nvml_handle(self):
        import pynvml as nv
        nv.nvmlInit()
        idx = self.device
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis and vis.split(",")[self.device].strip().isdigit():
            idx = int(vis.split(",")[self.device])
        self.nv = nv
        return nv.nvmlDeviceGetHandleByIndex(idx)

    def _nvml_sample(self):
        nv, h = self.nv, self.h
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                             float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)),
                             {n for n, bit in zip(self.NAMES, bits) if r & bit}))

    def _poll(self):
        while not self.stop.wait(0.01):
            try:
                self._nvml_sample()
            except Exception:
                return

    def __enter__(self):
        try:
            self.h = self._nvml_handle()
            self._nvml_sample()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nv = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) == 7 and p[0].replace(".", "").isdigit():
                self.samples.append((float(p[0]), float(p[1]) if p[1].replace(".", "").isdigit() else 0.0,
                                     {n for n, v in zip(self.NAMES, p[3:]) if v.lower() == "active"}))

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.thread.join(timeout=1)
            try:
                self._nvml_sample()  # the region's trailing edge (the step stream was just synchronised)
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [x[0] for x in self.samples]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": sorted(set().union(*(x[2] for x in self.samples))), "samples": len(self.samples),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


def load_lengths():
    rows = []
    with open(os.path.join(C3_DIR, "lengths.csv")) as fh:
        next(fh)
        for line in fh:
            a, b = line.strip().split(",")
            rows.append((int(a), int(b)))
    return rows


def m_require(entries, C, avg_out, min_total):
    """proj/src/memory.cpp:19-27: ceil(C * max(sum_r I_r + max(gen_r, avg_out), min_total_len))."""
    tot = sum(i + max(float(g), avg_out) for i, g in entries)
    return int(-(-max(tot, float(min_total)) * C // 1))


def watermark_decide(cur, req, pct=WATERMARK):
    """proj/src/memory.cpp:29-36 (scale_bytes_up applied twice for the down test)."""
    up = lambda b: int(-(-b * (100.0 + pct) // 100.0))  # noqa: E731
    rec = up(req)
    if cur < req:
        return "up", rec
    if up(rec) < cur:
        return "down", rec
    return "hold", rec


class Colocated:
    """The C3 node: eight instances, each with a full batch of 8, served in turns."""

    def __init__(self, device: int, seed: int = 7):
        import random

        from paper_2507_00507_b200.gpu import SHAPES, MeshGpu
        # the whole KV arena backed at open: no VMM driver call (each drains the device) while serving
        prev = os.environ.get("MESH_GPU_KV_PREALLOC_GB")
        os.environ["MESH_GPU_KV_PREALLOC_GB"] = prev or str(KV_POOL >> 30)
        try:
            self.g = MeshGpu(device, kv_pool_bytes=KV_POOL, prompt_seed=seed, lanes=LANES,
                             kv_granule_bytes=KV_GRANULE_MB << 20)
        finally:
            if prev is None:
                del os.environ["MESH_GPU_KV_PREALLOC_GB"]
        self.shapes = [SHAPES[m] for m in MODELS]
        self.rng = random.Random(seed)
        self.lengths = load_lengths()
        self.avg_out = sum(o for _, o in self.lengths) / len(self.lengths)  # avg_output_fixed
        self.next_rid = 0
        self.insts = []
        for iid, (m, shape) in enumerate(zip(MODELS, self.shapes)):
            # replicas of a model share one weight set (same model => same weights)
            self.g.create_instance(iid, shape, seed=1000 + MODELS.index(m))
            self.insts.append({"id": iid, "model": m, "shape": shape, "reqs": [], "pending": [], "kv": 0})
        self.clock = 0.0  # device-time clock (s) for SLO accounting
        self.mark0 = None  # clock value at timer mark 0: emissions are then read off the device timeline
        self.kv_grows = self.kv_shrinks = 0
        self.reset_counters()

    def kv_update(self, inst):
        """Re-size the instance's KV target by the reference's watermark rule."""
        s = inst["shape"]
        entries = [(r["I"], r["sched"]) for r in inst["reqs"] + inst["pending"]]
        req = m_require(entries, s.kv_bytes_per_token, self.avg_out, s.max_seq_len)
        act, rec = watermark_decide(inst["kv"], req)
        if act == "hold":
            return
        self.g.kv_resize(inst["id"], inst["kv"], rec)
        inst["kv"] = rec
        if act == "up":
            self.kv_grows += 1
        else:
            self.kv_shrinks += 1

    def new_request(self, inst):
        i, o = self.lengths[self.rng.randrange(len(self.lengths))]
        cap = inst["shape"].max_seq_len
        if i + o > cap:
            o = max(1, cap - i)
        r = {"rid": self.next_rid, "I": i, "O": o, "gen": 0, "sched": 0, "arrival": self.clock, "ok": True}
        self.next_rid += 1
        inst["pending"].append(r)
        self.kv_update(inst)

    def fill(self):
        for inst in self.insts:
            while len(inst["reqs"]) + len(inst["pending"]) < BATCH:
                self.new_request(inst)

    def plan_of(self, inst):
        """The instance's next step: a pending request is prefilled first (select_next's
        prefill-first rule), else the decode of its batch."""
        if inst["pending"]:
            return "prefill", [inst["pending"][0]]
        return "decode", list(inst["reqs"])

    def launch(self, inst, kind, reqs):
        if kind == "prefill":
            r = reqs[0]
            return self.g.step_async(inst["id"], prefill=r["rid"], prefill_len=r["I"], input_len=r["I"])
        return self.g.step_async(inst["id"], decode=[r["rid"] for r in reqs])

    def schedule_effects(self, inst, kind, reqs):
        """Host-side state the next plans depend on (known without waiting for the GPU)."""
        if kind == "prefill":
            r = inst["pending"].pop(0)
            r["sched"] = 1
            inst["reqs"].append(r)
            done = [r] if r["sched"] >= r["O"] else []
        else:
            for r in reqs:
                r["sched"] += 1
            done = [r for r in reqs if r["sched"] >= r["O"]]
        for r in done:
            inst["reqs"].remove(r)
            # completion: its blocks return now (stream-ordered after its last step on the
            # instance's lane), so the KV shrink of the watermark rule sees the schedule's state
            self.g.request_free(inst["id"], r["rid"])
            self.new_request(inst)

    def run(self, steps):
        """Launch `steps` steps asynchronously. Every instance keeps up to DEPTH steps
        queued on its own lane and gets its next step as soon as one of its steps
        retires, so each lane runs at its own pace (a round-robin issue order would
        hold fast lanes to the slowest lane's step time)."""
        from collections import deque
        DEPTH = 4
        q = [deque() for _ in self.insts]
        launches0 = self.g.stats()["kernel_launches"]
        issued = 0

        def issue(i):
            inst = self.insts[i]
            kind, reqs = self.plan_of(inst)
            q[i].append((self.launch(inst, kind, reqs), inst, kind, reqs))
            self.schedule_effects(inst, kind, reqs)

        if os.environ.get("MESH_BENCH_ISSUE") == "rr":  # A/B: round-robin issue, in-order retire, <= 32 in flight
            inflight = deque()
            for k in range(steps):
                inst = self.insts[k % len(self.insts)]
                kind, reqs = self.plan_of(inst)
                inflight.append((self.launch(inst, kind, reqs), inst, kind, reqs))
                self.schedule_effects(inst, kind, reqs)
                while len(inflight) > 32:
                    self.retire(inflight.popleft())
            while inflight:
                self.retire(inflight.popleft())
            return self.g.stats()["kernel_launches"] - launches0
        while issued < steps:
            # fill every lane's queue (fewest in flight first, then index)
            for i in sorted(range(len(self.insts)), key=lambda j: (len(q[j]), j)):
                if issued < steps and len(q[i]) < DEPTH:
                    issue(i)
                    issued += 1
            # retire finished steps; if none finished, wait for the oldest queued one
            progressed = False
            for i in range(len(q)):
                while q[i] and self.g.done(q[i][0][0]):
                    self.retire(q[i].popleft())
                    progressed = True
            if not progressed and issued < steps:
                # wait for ANY lane's head step (blocking on one ticket would let the other
                # lanes run dry behind a long prefill)
                time.sleep(5e-5)
        for i in range(len(q)):
            while q[i]:
                self.retire(q[i].popleft())
        return self.g.stats()["kernel_launches"] - launches0

    def retire(self, item):
        """Step finished: advance the device-time clock, account tokens against the SLO."""
        t, inst, kind, reqs = item
        self.g.wait(t)
        st = self.g.stats()
        if self.mark0 is not None and st["last_step_end_ms"] >= 0:
            emit = self.mark0 + st["last_step_end_ms"] / 1e3  # the step's end on the device timeline
        else:
            emit = self.clock + st["last_step_ms"] / 1e3      # no mark yet: steps back to back
        self.clock = max(self.clock, emit)
        busy = self.lane_busy.setdefault(inst["id"], [0.0, 0])
        busy[0] += st["last_step_ms"]
        busy[1] += 1
        if kind == "decode":
            s = inst["shape"]
            ctx = sum(r["I"] + r["gen"] for r in reqs)
            b = (s.weight_bytes_streamed + ctx * s.kv_bytes_per_token + len(reqs) * s.kv_bytes_per_token +
                 len(reqs) * s.d_model * 2)
            self.decode_bytes += b
            self.decode_kernel_ms += st["last_kernel_ms"]
            self.decode_steps += 1
            pm = self.per_model.setdefault(inst["model"], {"bytes": 0.0, "kernel_ms": 0.0, "launches": 0})
            pm["bytes"] += b
            pm["kernel_ms"] += st["last_kernel_ms"]
            pm["launches"] += 1
        else:
            self.prefill_steps += 1
            self.prefill_ms += st["last_step_ms"]
        for r in reqs:
            deadline = r["arrival"] + max(2.0, r["I"] / 512.0) + 0.25 * r["gen"]
            if emit > deadline + 1e-9:
                r["ok"] = False
            r["gen"] += 1
            self.tokens_all += 1
            self.tokens_ok += 1 if r["ok"] else 0
            if r["gen"] >= r["O"]:
                self.completed += 1
                self.violations += 0 if r["ok"] else 1

    def reset_counters(self):
        self.tokens_ok = self.tokens_all = self.completed = self.violations = 0
        self.decode_bytes = self.decode_kernel_ms = 0.0
        self.decode_steps = self.prefill_steps = 0
        self.prefill_ms = 0.0
        self.per_model = {}
        self.lane_busy = {}  # instance -> [sum of its steps' device time (ms), steps]
        self.kv_grows = self.kv_shrinks = 0


def ref_config(cfg_path: str) -> str:
    """The reference simulator's schema has no `runtime` section: a copy without it."""
    import tempfile
    with open(cfg_path) as fh:
        cfg = json.load(fh)
    cfg.pop("runtime", None)
    cfg["output"] = {"dir": tempfile.mkdtemp(prefix="mesh_ref_"), "event_log": False}
    path = os.path.join(cfg["output"]["dir"], "config.json")
    with open(path, "w") as fh:
        json.dump(cfg, fh)
    return path


def reference_simulator_sample(scale: int):
    """The reference's own CPU code (its simulator, oracle/_ref) on the C3 trace: 1 core."""
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_capture")
    if not os.path.exists(ref):
        return None
    out = subprocess.run([ref, "time", ref_config(os.path.join(C3_DIR, f"s{scale}", "config.json")), "5"],
                         cwd=ROOT, capture_output=True, text=True)
    if out.returncode != 0:
        return None
    r = json.loads(out.stdout.strip().splitlines()[-1])
    return {"simulated_tokens_per_cpu_s": r["tokens"] / r["best_s"], "cores": 1, "kind": "reference",
            "sample": f"reference simulator (oracle/_ref) on the C3 trace at load scale {scale}: "
                      f"{r['tokens']} virtual tokens, {r['events']} events, best of 5 = {r['best_s']:.4f} s",
            "note": "virtual-time tokens: the reference prices steps from tables and computes no tokens"}


class CpuColocated:
    """The C3 node on the host CPU: the batched CPU decode (oracle/cpu_decode.c)
    over the same eight instances x batch 8, instances in turn. Replicas of a
    model share its weights (one oracle model per size class, as on the GPU);
    each instance's batch starts at contexts I + U[0, O) drawn from the same
    length set as the GPU node's requests (KV declared resident, values zero:
    a decode step's cost depends on the context, not the values), and every
    step advances them by one token. Prefill is not run on the CPU (it would
    only lower the CPU number)."""

    def __init__(self, seed: int = 7):
        import dataclasses
        import random

        from oracle import llama_oracle as ora
        from paper_2507_00507_b200.gpu import SHAPES
        self.ora = ora
        rng = random.Random(seed)
        lengths = load_lengths()
        self.models = {}
        for m in dict.fromkeys(MODELS):
            shape = dataclasses.replace(SHAPES[m], max_seq_len=min(SHAPES[m].max_seq_len, CPU_MAX_SEQ))
            self.models[m] = ora.Oracle(shape, 1000 + MODELS.index(m))
        self.insts = []
        for m in MODELS:  # per-class sequences are shared by that class's replicas (memory)
            if any(x["model"] == m for x in self.insts):
                self.insts.append(next(x for x in self.insts if x["model"] == m))
                continue
            seqs, toks = [], []
            for b in range(BATCH):
                i, o = lengths[rng.randrange(len(lengths))]
                q = self.models[m].new_seq()
                q.set_len(i + rng.randrange(o))
                seqs.append(q)
                toks.append(ora.prompt_token(seed, b, 0, self.models[m].shape.vocab))
            self.insts.append({"model": m, "seqs": seqs, "toks": toks})
        self.k = 0
        self.threads = ora.threads()

    def mean_context(self):
        seen = {id(x): x for x in self.insts}.values()
        lens = [self.ora.C.cast(self.ora.C.c_void_p(q.h), self.ora.C.POINTER(self.ora.C.c_int))[0]
                for x in seen for q in x["seqs"]]
        return sum(lens) / len(lens)

    def step(self) -> int:
        inst = self.insts[self.k % len(self.insts)]
        self.k += 1
        for q in inst["seqs"]:  # a sequence at the end of its buffer restarts at a short context
            if self.ora.C.cast(self.ora.C.c_void_p(q.h), self.ora.C.POINTER(self.ora.C.c_int))[0] >= CPU_MAX_SEQ - 2:
                q.set_len(64)
        inst["toks"] = self.ora.feed_batch(self.models[inst["model"]], inst["seqs"], inst["toks"])
        return BATCH


def cpu_port_sample():
    """cpu_baseline: bounded sample (~CPU_SAMPLE_S) of C3 instance steps on the host CPU."""
    node = CpuColocated()
    ctx0 = node.mean_context()
    for _ in range(3):  # one step of each model class (warm)
        node.step()
    n_tok, n_steps, t0 = 0, 0, time.perf_counter()
    while n_steps < len(MODELS) or time.perf_counter() - t0 < CPU_SAMPLE_S:
        n_tok += node.step()
        n_steps += 1
    dt = time.perf_counter() - t0
    return {"value": n_tok / dt, "unit": UNIT, "cores": node.threads, "kind": "port",
            "sample": f"{n_steps} C3 instance steps ({MODELS} in turn, batch 8, mean context {ctx0:.0f} "
                      f"from the C3 length set) of the batched CPU decode (oracle/cpu_decode.c, fp32 math on "
                      f"bf16 weights, {node.threads} threads): {n_tok} tokens in {dt:.2f} s",
            "same_config": True}


def run_reference(args, d: Dist):
    """Reference arm: the CPU execution of the co-located C3 step on the box's host cores."""
    if d.rank != 0:
        return
    node = CpuColocated()
    ctx0 = node.mean_context()
    for _ in range(args.warmup):
        node.step()
    t0 = time.perf_counter()
    tokens = sum(node.step() for _ in range(args.steps))
    total = time.perf_counter() - t0
    value = tokens / total
    sim = reference_simulator_sample(E2E_SCALES[0])
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (random-init weights)",
            "impl": "reference",
            "config": {"workload": "C3: 8 co-located Llama-shaped instances [1.1B, 3B, 7B, 1.1B, 3B, 7B, 1.1B, 3B], "
                                   "batch 8 each, instances in turn (host CPU)",
                       "models": MODELS, "batch_per_instance": BATCH, "mean_context": ctx0,
                       "step": "one instance step: batched decode of its 8 requests"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": node.threads, "kind": "port",
                             "sample": f"{args.steps} C3 instance steps of oracle/cpu_decode.c (batched, "
                                       f"{node.threads} threads, mean context {ctx0:.0f})"},
            "reference_simulator": sim,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_e2e_scale(device: int, scale: int):
    """The C3 bursty trace at one load scale through llmmesh.h, wall-clock mode."""
    import tempfile

    from paper_2507_00507_b200 import control, gpu
    os.environ["MESH_GPU_LANES"] = str(LANES)  # the data plane under the control plane: one lane per instance
    os.environ.setdefault("MESH_GPU_KV_PREALLOC_GB", str(KV_PREALLOC_GB))  # physical KV granules created at open
    os.environ.setdefault("MESH_GPU_KV_GRANULE_MB", str(KV_GRANULE_MB))
    cfg = os.path.join(C3_DIR, f"s{scale}", "config.json")
    with control.Experiment(cfg) as exp:
        exp.out_dir(tempfile.mkdtemp(prefix="mesh_e2e_"))
        exp.attach_gpu([device], E2E_KV_POOL, gpu.LIB_PATH)
        exp.run()
        names = ["wall_s", "gpu.steps", "gpu.decode_tokens", "gpu.prefill_tokens", "gpu.h2d_bytes", "gpu.d2h_bytes",
                 "gpu.device_ms", "gpu.lane_busy_s", "slo_compliant_rate", "total_requests", "slo_compliant",
                 "slo_compliant_decode_tokens", "output_tokens", "gpu.kernel_launches", "gpu_instances_avg",
                 "gpu_instances_max", "gpu.instance_starts", "gpu.weight_cache_hits", "gpu.blocks_moved",
                 "gpu.swap_out_bytes", "gpu.migrations", "evictions", "run_length_s", "gpu.dp_ms.step",
                 "gpu.dp_ms.kv_resize", "gpu.dp_ms.instance_create", "gpu.host_ms.step_wait", "displacements",
                 "gpu_models_avg", "gpu_models_max"]
        m = {k: exp.metric(k) for k in names}
    m["scale"] = scale
    m["slo_tokens"] = m["slo_compliant_decode_tokens"] + m["slo_compliant"]  # + each compliant request's first token
    m["tokens_at_slo_per_s"] = m["slo_tokens"] / m["wall_s"]
    return m


FLEET_FUNCS = 32
FLEET_WINDOW = 30.0
FLEET_LOADS = [int(x) for x in os.environ.get("MESH_BENCH_FLEET_LOADS", "1,2,3").split(",")]


def fleet_scenario(n_nodes: int, k: float, seed: int = 4242, window: float = FLEET_WINDOW,
                   mem_gb: float = 150.0) -> str:
    """C5 restated for the fleet e2e: 32 functions cycling [1b, 3b, 7b] on n_nodes GPU
    nodes (node i -> device i), the acceptance overload generator's three phases
    (proj/tests/acceptance_main.cpp:462-488: 0.08, 0.28, then 0.8 for 6 hot functions
    and 0.03 for the rest, req/s per function) compressed into a 30 s window, every
    rate x k (k = per-GPU load units x n_nodes), defragmentation on, wall clock."""
    import random
    import tempfile
    d = tempfile.mkdtemp(prefix=f"mesh_fleet_n{n_nodes}_k{k}_")
    rng = random.Random(seed)
    rows = []
    for f in range(FLEET_FUNCS):
        fn = f"fn{f:02d}"
        for t0, t1, rate in ((0.0, 0.2, 0.08), (0.2, 0.6, 0.28), (0.6, 1.0, 0.8 if f < 6 else 0.03)):
            t = t0 * window
            while True:
                t += rng.expovariate(rate * k)
                if t >= t1 * window:
                    break
                rows.append((t, fn))
    rows.sort()
    with open(os.path.join(d, "trace.csv"), "w") as fh:
        fh.write("timestamp_s,function_id\n")
        for t, fn in rows:
            fh.write(f"{t:.6f},{fn}\n")
    with open(os.path.join(C3_DIR, "s1", "config.json")) as fh:
        cfg = json.load(fh)
    cfg["cluster"]["nodes"] = [{"class": "gpu", "count": n_nodes, "mem_gb": mem_gb}]
    cfg["models"]["assignment"] = [["1b", "3b", "7b"][f % 3] for f in range(FLEET_FUNCS)]
    cfg["workload"].update({"trace": os.path.join(d, "trace.csv"), "window_s": window,
                            "sample_functions": len({fn for _, fn in rows})})
    cfg["output"] = {"dir": os.path.join(d, "out"), "event_log": False}
    path = os.path.join(d, "config.json")
    with open(path, "w") as fh:
        json.dump(cfg, fh)
    return path


def run_fleet_load(devices, load: int):
    """One fleet run: len(devices) GPU nodes, per-GPU load `load`, one host event loop."""
    import tempfile

    from paper_2507_00507_b200 import control, gpu
    os.environ["MESH_GPU_LANES"] = str(LANES)
    os.environ.setdefault("MESH_GPU_KV_PREALLOC_GB", str(KV_PREALLOC_GB))
    os.environ.setdefault("MESH_GPU_KV_GRANULE_MB", str(KV_GRANULE_MB))
    n = len(devices)
    with control.Experiment(fleet_scenario(n, load * n)) as exp:
        exp.out_dir(tempfile.mkdtemp(prefix="mesh_fleet_out_"))
        exp.attach_gpu(list(devices), E2E_KV_POOL, gpu.LIB_PATH)
        exp.run()
        names = ["wall_s", "gpu.steps", "gpu.h2d_bytes", "gpu.d2h_bytes", "gpu.lane_busy_s", "slo_compliant_rate",
                 "total_requests", "slo_compliant", "slo_compliant_decode_tokens", "output_tokens",
                 "gpu_instances_avg", "gpu_instances_max", "gpu_nodes_used", "gpu_nodes_avg", "gpu.instance_starts",
                 "gpu_models_avg", "gpu_models_max",
                 "gpu.migrations", "gpu.migrate_bytes", "gpu.swap_out_bytes", "displacements", "evictions"]
        m = {k: exp.metric(k) for k in names}
    m["load_per_gpu"] = load
    m["slo_tokens"] = m["slo_compliant_decode_tokens"] + m["slo_compliant"]
    m["tokens_at_slo_per_s"] = m["slo_tokens"] / m["wall_s"]
    return m


def run_fleet(n: int):
    """C5 fleet e2e (rank 0 drives devices 0..n-1 from one host loop): capacity sweep
    over per-GPU load; the headline is the highest load with compliance >= 0.99."""
    runs = [run_fleet_load(list(range(n)), k) for k in FLEET_LOADS]
    ok = [r for r in runs if r["slo_compliant_rate"] >= 0.99]
    head = max(ok, key=lambda r: r["load_per_gpu"]) if ok else min(runs, key=lambda r: r["load_per_gpu"])
    steps = max(1.0, head["gpu.steps"])
    return {"value": head["slo_tokens"] / head["wall_s"], "unit": UNIT,
            "h2d_bytes_per_step": head["gpu.h2d_bytes"] / steps, "d2h_bytes_per_step": head["gpu.d2h_bytes"] / steps,
            "workload": f"C5: fleet of 32 functions [1b, 3b, 7b] bin-packed over {n} B200 nodes (node i -> device i) "
                        "by the control plane, one host event loop, wall clock",
            "capacity_load_per_gpu": head["load_per_gpu"] if ok else None,
            "slo_compliant_rate": head["slo_compliant_rate"], "wall_s": head["wall_s"],
            "models_per_gpu": {"time_avg": head["gpu_instances_avg"], "max": head["gpu_instances_max"],
                               "distinct_models_time_avg": head["gpu_models_avg"],
                               "distinct_models_max": head["gpu_models_max"],
                               "gpu_nodes_used": head["gpu_nodes_used"]},
            "sweep": [{k: r[k] for k in ("load_per_gpu", "total_requests", "slo_compliant_rate", "tokens_at_slo_per_s",
                                         "wall_s", "gpu_instances_avg", "gpu_instances_max", "gpu_nodes_used",
                                         "gpu.instance_starts", "gpu.migrations", "gpu.migrate_bytes",
                                         "displacements", "evictions")} for r in runs],
            "trace": "acceptance overload generator (32 functions, three phases) in a 30 s window, rates x "
                     "(per-GPU load x n GPUs)",
            "api": "llmmesh.h llm_experiment_run + llm_experiment_attach_gpu(devices 0..n-1), runtime.clock = wall"}


def run_c4(device: int):
    try:
        return _run_c4(device)
    except Exception as e:  # wall-clock decisions are timing-dependent: the reference's eviction
        # ping-pong defect can end a C4 run; report it instead of failing the bench
        return {"error": str(e)}


def _run_c4(device: int):
    """C4 beside the headline (scenarios/c4_b200: 7B + 13B under KV pressure, wall clock):
    evictions swap running requests' KV to pinned host memory inside the timed region."""
    import tempfile

    from paper_2507_00507_b200 import control, gpu
    os.environ["MESH_GPU_LANES"] = str(LANES)
    os.environ.setdefault("MESH_GPU_SWAP_POOL_MB", "4096")
    with control.Experiment(os.path.join(ROOT, "scenarios", "c4_b200", "config.json")) as exp:
        exp.out_dir(tempfile.mkdtemp(prefix="mesh_c4_"))
        exp.attach_gpu([device], 48 << 30, gpu.LIB_PATH)
        exp.run()
        names = ["wall_s", "slo_compliant_rate", "total_requests", "slo_compliant", "slo_compliant_decode_tokens",
                 "evictions", "pingpong_drops", "gpu.swap_out_bytes", "gpu.swap_in_bytes", "gpu.steps", "gpu.decode_tokens",
                 "gpu_instances_avg",
                 "gpu.blocks_moved"]
        m = {k: exp.metric(k) for k in names}
    m["tokens_at_slo_per_s"] = (m["slo_compliant_decode_tokens"] + m["slo_compliant"]) / m["wall_s"]
    m["workload"] = ("C4: 7B + 13B functions on a 44 GB node (KV pressure, output estimator fixed low): "
                     "ensure_kv_capacity evicts, the data plane swaps KV to pinned host memory and back")
    return m


def run_e2e(device: int, d: Dist, scales):
    """Load sweep: among the scales whose wall-clock compliance is >= 0.99, the one with the most SLO
    tokens per second is the reported point (past saturation a heavier load only stretches the run)."""
    runs = []
    for k in scales:
        d.barrier()
        runs.append(run_e2e_scale(device, k))
    ok = [r for r in runs if r["slo_compliant_rate"] >= 0.99]
    head = max(ok, key=lambda r: r["tokens_at_slo_per_s"]) if ok else min(runs, key=lambda r: r["scale"])
    wall_max = d.reduce(head["wall_s"], "max")
    tok_sum = d.reduce(head["slo_tokens"], "sum")
    steps = max(1.0, head["gpu.steps"])
    return {"value": tok_sum / wall_max, "unit": UNIT,
            "h2d_bytes_per_step": head["gpu.h2d_bytes"] / steps, "d2h_bytes_per_step": head["gpu.d2h_bytes"] / steps,
            "capacity_scale": head["scale"] if ok else None,
            "capacity_rule": "most SLO tokens/s among load scales with wall-clock slo_compliant_rate >= 0.99",
            "max_compliant_scale": max(r["scale"] for r in ok) if ok else None,
            "slo_compliant_rate": head["slo_compliant_rate"], "wall_s": wall_max,
            "models_per_gpu": {"time_avg": head["gpu_instances_avg"], "max": head["gpu_instances_max"],
                               "distinct_models_time_avg": head["gpu_models_avg"],
                               "distinct_models_max": head["gpu_models_max"],
                               "note": "model instances resident per GPU (replicas of a model share its weights)"},
            "lane_busy_frac": head["gpu.lane_busy_s"] / (LANES * head["wall_s"]) if head["wall_s"] else None,
            "sweep": [{k: r[k] for k in ("scale", "total_requests", "slo_compliant_rate", "tokens_at_slo_per_s",
                                         "wall_s", "gpu_instances_avg", "gpu_instances_max", "gpu.steps",
                                         "gpu.instance_starts", "gpu.weight_cache_hits", "gpu.blocks_moved",
                                         "gpu.swap_out_bytes", "evictions", "gpu.dp_ms.step", "gpu.dp_ms.kv_resize",
                                         "gpu.dp_ms.instance_create", "gpu.host_ms.step_wait", "gpu.lane_busy_s")}
                      for r in runs],
            "trace": "scenarios/c3_b200/s{K}: acceptance overload generator's three phases (0.08, 0.28, "
                     "0.8 hot / 0.03 req/s per function) in a 30 s window, rates x K",
            "tables": "measured B200 tables + CostParams (admission); completions on CUDA events",
            "api": "llmmesh.h llm_experiment_run + llm_experiment_attach_gpu, runtime.clock = wall"}


class HostProfile:
    """MESH_BENCH_HOSTPROF=1: host seconds spent in each MeshGpu call of the timed loop
    (stderr), to tell host-issue gaps from device time."""

    def __init__(self, node):
        self.acc = {}
        g = node.g
        for name in ("step_async", "wait", "done", "stats", "kv_resize", "request_free"):
            f = getattr(g, name)

            def wrap(*a, _f=f, _n=name, **k):
                t0 = time.perf_counter()
                try:
                    return _f(*a, **k)
                finally:
                    e = self.acc.setdefault(_n, [0.0, 0])
                    e[0] += time.perf_counter() - t0
                    e[1] += 1
            setattr(g, name, wrap)

    def report(self, wall):
        tot = sum(v[0] for v in self.acc.values())
        print(json.dumps({"host_wall_s": round(wall, 3), "in_calls_s": round(tot, 3),
                          "calls": {k: [round(v[0], 4), v[1], round(1e6 * v[0] / max(1, v[1]), 1)]
                                    for k, v in sorted(self.acc.items())}}), file=sys.stderr)


def run_ours(args, d: Dist):
    device = d.local
    hbm, peak_kind = peaks()
    node = Colocated(device)
    node.k = 0
    node.g.sync()
    node.g.timer_mark(0)  # emissions read off the device timeline from the first admission on
    node.mark0 = 0.0
    node.fill()
    # initial admissions: every instance prefills its batch (untimed)
    node.run(len(MODELS) * BATCH)
    node.run(args.warmup * len(MODELS))
    node.g.sync()
    node.reset_counters()
    d.barrier()
    with Clocks(device) as clk:
        node.g.sync()
        node.g.timer_mark(0)
        node.mark0 = node.clock
        profiler_region(True)
        hp = HostProfile(node) if os.environ.get("MESH_BENCH_HOSTPROF") else None
        w0 = time.perf_counter()
        launches = node.run(args.steps)
        host_wall = time.perf_counter() - w0
        if hp:
            hp.report(host_wall)
        profiler_region(False)
        node.g.timer_mark(1)
        node.g.sync()
        dev_s = node.g.timer_elapsed(0, 1) / 1e3
    wall_max = d.reduce(dev_s, "max")
    tok_ok = d.reduce(float(node.tokens_ok), "sum")
    value = tok_ok / wall_max
    # Decode launches of the eight lanes overlap, so a launch's own duration is not the
    # time the node spends per launch: achieved = algorithmic decode bytes of every
    # launch over the timed device span (prefill steps inside the span make it a lower
    # bound); the single-launch figure (bytes / the launch's own CUDA-event time, on
    # its lane's SM quota) is kept beside it.
    per_launch = node.decode_bytes / (node.decode_kernel_ms / 1e3) / 1e9 if node.decode_kernel_ms else 0.0
    achieved = node.decode_bytes / dev_s / 1e9 if dev_s else 0.0
    quotas = [node.g.instance_lane(i["id"])[1] for i in node.insts]
    g_stats = node.g.stats()
    node.g.close()  # frees the node's HBM for the e2e leg
    if args.no_e2e:
        e2e = None
    elif d.ws == 1:
        e2e = run_e2e(device, d, E2E_SCALES)
        e2e["c4"] = run_c4(device)
    else:
        # the fleet: rank 0 drives every device through the control plane's placement
        # (one host event loop, peer access between the devices); the other ranks wait
        d.barrier(host=True)
        e2e = None
        if d.rank == 0:
            from paper_2507_00507_b200 import gpu
            if gpu.lib().mesh_gpu_device_count() >= d.ws:
                e2e = run_fleet(d.ws)
            else:  # this rank sees only its own GPU (per-rank CUDA_VISIBLE_DEVICES): one node
                e2e = run_e2e(device, Solo(), E2E_SCALES)
                e2e["note"] = "fleet skipped: rank 0 sees fewer GPUs than ranks; single-node C3 e2e"
        d.barrier(host=True)
    if d.rank != 0:
        return
    cpu = cpu_port_sample() if d.ws == 1 and not args.no_cpu else None
    sim = reference_simulator_sample(E2E_SCALES[0]) if d.ws == 1 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(prof):  # ncu DRAM bytes per launch per model, weighted by this run's launch mix
        with open(prof) as fh:
            per = json.load(fh).get("per_model", {})
        n = sum(v["launches"] for v in node.per_model.values())
        if per and n and all(m in per for m in node.per_model):
            traffic = sum(v["launches"] * per[m]["dram_bytes"] for m, v in node.per_model.items()) / n
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": d.ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, synthetic prompts)",
        "config": {"workload": "C3: 8 co-located Llama-shaped instances [1.1B, 3B, 7B, 1.1B, 3B, 7B, 1.1B, 3B] on "
                               "one B200, batch 8 each, shared VMM KV pool with watermark grow/shrink",
                   "models": MODELS, "batch_per_instance": BATCH, "step": "one instance step (decode of its batch "
                   "or prefill of a newly admitted request); every instance keeps <= 4 steps queued on its own "
                   f"execution lane ({LANES} lanes, SM quotas in proportion to streamed weight bytes), so "
                   "co-located instances step concurrently",
                   "lane_sm_quotas": quotas,
                   "l2": "weights 53 GB + KV streamed per 8-step round >> 126 MB L2 (no flush needed)",
                   "slo_compliant_tokens": int(node.tokens_ok), "tokens": int(node.tokens_all),
                   "completed_requests": node.completed, "slo_violations": node.violations,
                   "decode_steps": node.decode_steps, "prefill_steps": node.prefill_steps,
                   "kv_grows": node.kv_grows, "kv_shrinks": node.kv_shrinks,
                   "kv_blocks_moved": g_stats["blocks_moved"],
                   "lane_busy_frac": {str(i): round(v[0] / (1e3 * dev_s), 3) for i, v in sorted(node.lane_busy.items())},
                   "lane_steps": {str(i): v[1] for i, v in sorted(node.lane_busy.items())},
                   "prefill_step_ms_avg": round(node.prefill_ms / max(1, node.prefill_steps), 2),
                   "parallelism": f"{d.ws} independent co-located nodes"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm if hbm else None, "traffic": traffic,
                     "traffic_basis": "ncu dram__bytes_read+write per decode launch per model "
                                      "(profiles/decode_traffic.json), weighted by this run's launch mix",
                     "kernel": "decode_kernel (persistent, TMA-ring), one launch per lane step",
                     "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": node.decode_bytes / max(1, node.decode_steps),
                     "launches": node.decode_steps,
                     "achieved_basis": "sum of decode launches' algorithmic bytes / timed device span "
                                       "(lanes overlap; prefill steps in the span make this a lower bound)",
                     "per_launch_gbs": per_launch,
                     "per_launch_note": "bytes / the launch's own CUDA-event time on its lane's SM quota",
                     "per_model": {m: {"launches": v["launches"], "gbs_per_launch": v["bytes"] / (v["kernel_ms"] / 1e3) / 1e9,
                                       "ms_per_launch": v["kernel_ms"] / max(1, v["launches"])}
                                   for m, v in node.per_model.items()}},
        "cpu_baseline": cpu,
        "reference_simulator": sim,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


def main():
    os.chdir(ROOT)  # scenario configs use repo-relative paths
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    d = Dist()
    try:
        if args.impl == "reference":
            run_reference(args, d)
        else:
            run_ours(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
