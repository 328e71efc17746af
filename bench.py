#!/usr/bin/env python
"""PULSE encode+apply benchmark (BASELINE.json metric: "encode+apply weight GB/s
(frac. of HBM peak) at 1/2/4/8 B200; patch MB").

One step = one pass of the hot path over the configured state dict:
  encode  K1 diff+compaction -> [NCCL size exchange] -> K2 index coding / PULP body
          -> D2H of the entry table (the PULP header fields)
  apply   parse + validate + scatter the body into resident weights, in place.
Steps alternate direction (prev->curr, then curr->prev) so every step does the
same work on the same resident weights.  value = 2*d bytes of weights per step
/ step time, whole job (all ranks), max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload qwen2.5-7b]
  python bench.py --impl reference ...   # the reference CPU path on host cores
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

from paper_2602_03839_b200.shapes import numel, shard, workload  # noqa: E402

REPR_NAMES = {0: "COO_DOWNSCALED", 1: "COO_INT32", 2: "FLAT_INT32"}
METRIC = "encode+apply weight GB/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pulse", choices=["pulse", "reference"])
    ap.add_argument("--workload", default="qwen2.5-7b")
    ap.add_argument("--sparsity", type=float, default=0.99)
    ap.add_argument("--cluster-width", type=int, default=64)
    ap.add_argument("--repr", type=int, default=0, choices=[0, 1, 2])
    ap.add_argument("--seed", type=int, default=1002)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replays")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-elems", type=int, default=480_000_000)
    return ap.parse_args()


READ_STREAM_GBS = 7400.0  # profiles/r2a_bw_probe.txt: best read-only streaming kernel on B200


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------------------------------
# clocks during the timed region
# ------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region: NVML
    polled every 5 ms from a thread (nvidia-smi -lms 100 as a fallback)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.dev = device_index
        self.period = period_s
        self.sm, self.mx, self.reasons = [], None, set()
        self.proc = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self._nvml_index(nv))
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self.stop.is_set():
                    self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    r = int(get_reasons(h))
                    for name, bit in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(name)
                    time.sleep(self.period)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.mode = "nvml"
        except Exception:
            self.mode = "nvidia-smi"
            self._start_smi()
        return self

    def _nvml_index(self, nv):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",")]
            if self.dev < len(ids) and ids[self.dev].isdigit():
                return int(ids[self.dev])
        return self.dev

    def _start_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + fields,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def read():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                try:
                    self.sm.append(float(parts[0]))
                    self.mx = float(parts[1])
                except (ValueError, IndexError):
                    continue
                for name, v in zip(names, parts[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(name)
        self.t = threading.Thread(target=read, daemon=True)
        self.t.start()

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif getattr(self, "t", None):
            self.t.join(timeout=1)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": self.mode}


# ------------------------------------------------------------------------------------------
# reference CPU path (oracle/_ref: the unmodified reference headers), host cores
# ------------------------------------------------------------------------------------------
def numpy_pair(shapes, sparsity, cluster, seed):
    """Sample input for the CPU legs: log-normal bf16 weights and clustered
    half-density LSB flips (the reference generator's knobs, numpy RNG)."""
    rng = np.random.default_rng(seed)
    prev, curr = [], []
    for shp in shapes:
        n = numel(shp)
        x = np.exp(np.log(0.0117) + rng.standard_normal(n, dtype=np.float32)).astype(np.float32)
        x[rng.random(n, dtype=np.float32) < 0.5] *= -1
        u = x.view(np.uint32)
        b = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)  # RNE to bf16
        c = b.copy()
        n_change = int(round((1 - sparsity) * n))
        starts = rng.integers(0, n, max(1, 2 * n_change // max(1, cluster)))
        pos = (starts[:, None] + np.arange(cluster)[None, :]).ravel()
        pos = pos[(pos < n) & (rng.random(pos.size) < 0.5)]
        pos = np.unique(pos)[:n_change]
        c[pos] ^= 1
        prev.append(b)
        curr.append(c)
    return prev, curr


def time_reference(names, shapes, prev, curr, repr_, steps, warmup):
    """Times the reference's own hot path on one core: encode (patch.hpp:264,
    incl. its SHA-256 target hash) + write_patch_bytes + read_patch_bytes +
    decode(verify=false) (patch.hpp:309).  Returns per-step seconds + parts."""
    from oracle.oracle import Checkpoint, Tensor, reference, IDENTITY
    R = reference()
    hp = R.ckpt_handle(Checkpoint(0, [Tensor(n, s, a) for n, s, a in zip(names, shapes, prev)]))
    hc = R.ckpt_handle(Checkpoint(1, [Tensor(n, s, a) for n, s, a in zip(names, shapes, curr)]))
    try:
        per, parts = [], []
        for k in range(warmup + steps):
            a, b = (hp, hc) if k % 2 == 0 else (hc, hp)
            t, nbytes, changes = R.time_step(a, b, repr_, IDENTITY, verify=False)
            if k >= warmup:
                per.append(sum(t[x] for x in ("encode", "write", "read", "decode")))
                parts.append(t)
        return per, parts, nbytes, changes
    finally:
        R.L.ref_ckpt_free(hp)
        R.L.ref_ckpt_free(hc)


def cpu_sample(tensors, target_elems):
    """A bounded, representative slice of the workload: whole tensors in name
    order starting after the embeddings, up to ~target_elems elements."""
    picked, total = [], 0
    start = 2 if len(tensors) > 3 else 0
    for name, shp in tensors[start:]:  # consecutive in name order (FLAT gaps continue across them)
        n = numel(shp)
        if total and total + n > target_elems:
            break
        picked.append((name, shp))
        total += n
    return picked, total


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    tensors = workload(args.workload)
    picked, total = cpu_sample(tensors, args.cpu_sample_elems)
    names, shapes = [n for n, _ in picked], [s for _, s in picked]
    prev, curr = numpy_pair(shapes, args.sparsity, args.cluster_width, args.seed)
    per, parts, nbytes, changes = time_reference(names, shapes, prev, curr, args.repr, args.steps, args.warmup)
    sec = statistics.mean(per)
    value = 2 * total / sec / 1e9
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u16 (bf16 bit patterns)",
        "data": "synthetic (numpy log-normal bf16, clustered LSB flips)",
        "config": {"workload": args.workload, "sample_tensors": len(picked), "sample_elements": total,
                   "sparsity": args.sparsity, "cluster_width": args.cluster_width,
                   "representation": REPR_NAMES[args.repr], "codec": "identity"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "reference",
                         "sample": f"{len(picked)} tensors / {total} elements of {args.workload}",
                         "parts_s": {k: round(statistics.mean(p[k] for p in parts), 4) for k in parts[0]}},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "patch_mb": round(nbytes / 1e6, 3), "changes": changes,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# the PULSE arm
# ------------------------------------------------------------------------------------------
def run_pulse(args):
    import torch
    import torch.distributed as dist

    from paper_2602_03839_b200 import device as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL_DEBUG is left as the launcher set it (its INIT lines confirm the ranks);
        # NCCL's log goes to stderr so rank 0's stdout stays the one JSON line
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    from paper_2602_03839_b200.shard import ShardedPulse

    tensors = workload(args.workload)
    d_total = sum(numel(s) for _, s in tensors)
    sp = ShardedPulse(tensors, max_change_frac=(1 - args.sparsity) * 1.02)
    mine = sp.mine
    sizes = sp.sizes
    D_el = sum(sizes)
    assert all(n % 8 == 0 for n in sizes), "tensors must keep 16-byte alignment in the arena"

    # ---- resident snapshots (synthetic, generated on device) ----------------------------
    prev = torch.empty(max(8, D_el), dtype=torch.int16, device=dev)
    curr = torch.empty_like(prev)
    w = torch.empty_like(prev)
    D.synth_base(prev, seed=args.seed + 7919 * rank)
    D.synth_mutate(prev, curr, args.sparsity, args.cluster_width, seed=args.seed + 104729 * rank) if D_el else 0
    w.copy_(prev)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    views = lambda buf: [buf[int(offs[i]):int(offs[i + 1])] for i in range(len(sizes))]
    sp.bind(0, views(prev))
    sp.bind(1, views(curr))
    sp.bind(2, views(w))
    patch = sp.new_patch(args.repr)
    stream = torch.cuda.current_stream()

    ev = {k: [] for k in ("s0", "s1", "a0", "a1")}
    state = {"body": 0, "changes": 0}
    # steps actually executed on the device (incremented inside every step and graph
    # replay): the timed loop must have run exactly K steps, not merely left W where it was
    replays = torch.zeros(1, dtype=torch.int64, device=dev)

    def step(k, record=False):
        """scan -> (all-gather summaries, K2, size exchange, FLAT carry) -> apply:
        entirely stream-ordered on the device, no host round trip."""
        cs, ps = (1, 0) if k % 2 == 0 else (0, 1)
        if record:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        sp.plan.scan(cs, ps, summary_out=sp.send)
        if record:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
        sp.emit_async(patch)
        if record:
            a0 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
        sp.apply_async(2, patch)
        sp.join()  # the size exchange (side stream) belongs to the step
        replays.add_(1)
        if record:
            a1 = torch.cuda.Event(enable_timing=True)
            a1.record(stream)
            ev["s0"].append(e0); ev["s1"].append(e1); ev["a0"].append(a0); ev["a1"].append(a1)

    def check_step():
        """Host check of the last step's encode and apply results (outside timing)."""
        patch.fetch()
        if patch.status != 0:
            patch.raise_for_status([n for n, _ in mine])
        res = D.parse_result(sp.apply_res)
        if int(res["status"]) != 0:
            raise RuntimeError(f"apply failed: {res}")
        state["body"] = patch.body_bytes
        state["changes"] = patch.n_changes
        if world > 1 and not os.environ.get("PULSE_SKIP_SIZE_EXCHANGE"):  # the size exchange saw this rank's section
            torch.cuda.synchronize()
            dist.barrier()  # every rank's peer stores of its sizes have landed
            bb, _, st = sp.exchanged_sizes()
            if int(bb[rank]) != patch.body_bytes or any(int(x) != 0 for x in st):
                raise RuntimeError(f"size exchange mismatch: {bb} {st}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for k in range(args.warmup):
        step(k)
        check_step()
    # W must equal prev again before the timed loop starts on an even step
    if args.warmup % 2 == 1:
        step(args.warmup)
        check_step()
    barrier()
    # per-phase times (encode = scan, apply) from one eager pass over `steps` steps
    for k in range(args.steps):
        step(k, record=True)
    barrier()
    check_step()
    # the timed loop replays the step as a CUDA graph (one per direction: the two
    # snapshot slots swap), launch overhead off the host; eager launches if capture fails
    graphs = None
    if not args.no_graph:
        try:
            graphs = []
            for k in (0, 1):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    step(k)
                graphs.append(g)
            for k in (0, 1):  # the capture recorded, not ran: run both once, W is back at prev
                graphs[k].replay()
            torch.cuda.synchronize()
            check_step()
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] graph capture unavailable ({type(exc).__name__}: {exc}); timing eager launches",
                  file=sys.stderr)
            graphs = None
            torch.cuda.synchronize()
    barrier()
    replays_before = int(replays.item())
    stream = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        t0.record(stream)
        for k in range(args.steps):
            if graphs:
                graphs[k % 2].replay()
            else:
                step(k)
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    check_step()
    ms = t0.elapsed_time(t1) / args.steps
    used_graph = bool(graphs)
    graphs = None  # release the graphs (and anything they reference) before teardown
    scan_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev["s0"], ev["s1"]))
    apply_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev["a0"], ev["a1"]))
    emit_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev["s1"], ev["a0"]))

    # correctness: after the timed loop W must equal the last step's target, and
    # two more (untimed) steps must each land exactly on theirs
    ok = bool(torch.equal(w, prev if args.steps % 2 == 0 else curr))
    ran = int(replays.item()) - replays_before
    ok = ok and ran == args.steps
    for k in (args.steps, args.steps + 1):
        step(k)
        check_step()
        torch.cuda.synchronize()
        ok = ok and bool(torch.equal(w, curr if k % 2 == 0 else prev))

    t_ms = torch.tensor([ms, scan_ms, apply_ms, float(not ok), emit_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        tot = torch.tensor([float(state["body"]), float(state["changes"])], dtype=torch.float64, device=dev)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        body_total, changes_total = tot.tolist()
    else:
        body_total, changes_total = float(state["body"]), float(state["changes"])
    ms_max, scan_max, apply_max, bad, emit_max = t_ms.tolist()

    e2e = None
    if not args.no_e2e:
        if world == 1:
            e2e = run_e2e(args, mine, prev, curr, views, world, rank)
        else:
            # the reference operation's target_hash is ONE SHA-256 over the whole state dict in
            # name order (sha256.hpp:93-116); it does not shard, so the end-to-end number is
            # reported for the single-GPU run only
            e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                   "note": "end to end is measured at N=1: encode's whole-dict target hash is one sequential "
                           "SHA-256 and does not shard"}

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, parity = cpu_baseline_and_parity(args, mine, prev, curr, offs, sp, patch, step, check_step)

    if rank == 0:
        peak, peak_kind = measured_peaks()
        value = 2 * d_total / (ms_max / 1e3) / 1e9
        # dominant kernel K1: its algorithmic bytes are the two snapshots it reads
        # (4 B/elem); the 6 B/change K1->K2 intermediate it writes is overhead, reported beside it
        k1_bytes = 4 * D_el
        k1_gbs = k1_bytes / (scan_ms / 1e3) / 1e9
        k1_moved = 4 * D_el + 6 * state["changes"]
        # our launches per step: K1 (k1_tma, k1_deferred [graph: k_set_cond; K1b runs only if a ticket
        # was deferred], k1_finalize); K2 (COO: optimistic k2_layout + k2_emit, then
        # k2_scan_escapes / k2_layout / k2_emit that return at once unless an escape was seen; int32:
        # k2_layout, k2_emit); FLAT carry [sharded FLAT only]; apply (d_layout, f_stream agg, f_range_scan,
        # f_pass validate, its full re-check (exits at once unless a check failed), f_stream scatter,
        # d_clear_status, general-path kernels that exit at once on the fast path [COO: d_rows,
        # d_col_layout, d_cols, d_assemble; int32: d_fixed], d_scatter, d_finalize).
        # Replayed graphs: every idle path sits in a conditional node, one k_set_cond each instead.
        if used_graph:
            n_emit = 3 if args.repr == 0 else 2
            n_apply = 8
        else:
            n_emit = 5 if args.repr == 0 else 2
            n_apply = 13 if args.repr == 0 else 10
        n_carry = 1 if (world > 1 and args.repr == 2) else 0
        # N > 1: the size table goes out by one peer-store kernel (k_store_to_peers) per step
        # unless the NCCL fallback is in use (its kernels are not ours)
        n_peer = 1 if (world > 1 and getattr(sp, "_peer_ptrs", None) is not None
                       and not os.environ.get("PULSE_SKIP_SIZE_EXCHANGE")) else 0
        if world > 1 and args.repr == 2 and getattr(sp, "_sum_ptrs", None) is not None:
            n_peer += 2  # k_peer_post + k_peer_wait (FLAT summaries over NVLink)
        if world > 1:
            print(f"[bench] size table: {'NVLink peer stores' if sp._peer_ptrs is not None else 'NCCL all-gather'}",
                  file=sys.stderr)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u16 (bf16 bit patterns; integer/bitwise path)",
            "data": "synthetic (device log-normal bf16, clustered half-density LSB flips)",
            "config": {"workload": args.workload, "tensors": len(tensors), "elements": d_total,
                       "sparsity": args.sparsity, "cluster_width": args.cluster_width,
                       "representation": REPR_NAMES[args.repr], "codec": "identity (device body)",
                       "parallelism": f"tensor-shard x{world}" if world > 1 else "single GPU",
                       "launch": "cuda-graph replay" if used_graph else "eager",
                       "l2": f"inputs {4 * d_total / 1e9:.1f} GB per step >> 126 MB L2 (no flush needed)"},
            # the step against the HBM roofline (north_star: bytes read + written / peak), algorithmic
            # bytes per SURVEY §8(d): encode 4d + P_idx + 2n (snapshots in, patch body out), apply
            # P_idx + 2n (patch in) + 2n (scattered writes); the K1->K2 intermediate is not counted
            "frac_of_hbm": round((4 * d_total + 2 * body_total + 2 * changes_total) / (ms_max / 1e3) / 1e9
                                 / (peak * world), 4),
            "step_bytes": int(4 * d_total + 2 * body_total + 2 * changes_total),
            "weight_gbs_frac_of_peak": round(value / (peak * world), 4),
            "encode_ms": round(scan_max, 4), "apply_ms": round(apply_max, 4),
            "patch_mb": round(body_total / 1e6, 3), "changes": int(changes_total),
            "roofline": {"kernel": "k1_diff_compact", "bound": "hbm", "achieved": round(k1_gbs, 2),
                         "peak": peak, "unit": "GB/s", "frac": round(k1_gbs / peak, 4),
                         "traffic": profiled_traffic(args, world),
                         "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": k1_bytes,
                         "bytes_moved_per_launch": k1_moved,
                         "frac_incl_intermediate": round(k1_moved / (scan_ms / 1e3) / 1e9 / peak, 4),
                         # the measured peak is a copy (half read, half write); K1 only reads (+0.2% writes),
                         # and a read-only stream runs faster on B200: best of the read probe in
                         # profiles/r2a_bw_probe.txt (tools/bw_probe.cu, 30.5 GB read, 7.40 TB/s)
                         "read_stream_peak": READ_STREAM_GBS,
                         "frac_of_read_stream": round(k1_gbs / READ_STREAM_GBS, 4)},
            # every phase against the peak of the GPUs doing it (eager pass, CUDA events on the launching
            # stream, max over ranks); whole-job bytes per SURVEY 8(d): K2 reads the K1 intermediate
            # (6 B/change) and writes the body; apply reads the body and writes 2 B per change (scattered)
            "phases": {k: {"ms": round(t, 4), "bytes": int(b), "frac": round(b / (t / 1e3) / 1e9 / (peak * world), 4)}
                       for k, t, b in (("k1_scan", scan_max, 4 * d_total + 6 * changes_total),
                                       ("k2_emit", emit_max, 6 * changes_total + body_total),
                                       ("apply", apply_max, body_total + 2 * changes_total))},
            "gpu_launches": (3 + n_emit + n_carry + n_peer + n_apply) * args.steps,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity_vs_reference": parity,
            "verified": not bool(bad),
            "verified_detail": "after the timed loop W equals the last step's target, the device step counter "
                               "advanced by exactly `steps`, and two further steps each land exactly on theirs",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        if used_graph:
            # NCCL communicators captured in CUDA graphs: process-group teardown can
            # block on them, so leave without it once every rank is done
            sys.stdout.flush()
            sys.stderr.flush()
            os._exit(0)
        dist.destroy_process_group()
    return 0


def cpu_baseline_and_parity(args, mine, prev, curr, offs, sp, patch, step, check_step):
    """The reference CPU path timed on the SAME bytes the GPU encoded (a bounded
    sample of whole tensors, D2H from the device snapshots), and the reference's
    PULP blobs for those tensors byte-compared with their sections of the device
    patch body.

    FLAT_INT32: the sample's first changed tensor starts its own gap stream in the
    reference (absolute first index) while in the full patch it continues from the
    previous changed tensor; that one u32 is checked against
    numel(previous changed tensor) - its last changed index + the first index."""
    import torch

    from oracle.oracle import Checkpoint, Tensor, reference

    picked, total = cpu_sample(mine, args.cpu_sample_elems)
    names = [n for n, _ in picked]
    i0 = [n for n, _ in mine].index(names[0])
    i1 = i0 + len(picked)
    assert [n for n, _ in mine[i0:i1]] == names
    # one more step in the prev -> curr direction: the patch is then curr vs prev
    step(0)
    check_step()
    patch.fetch()

    def host(buf):
        a = buf[int(offs[i0]):int(offs[i1])].cpu().numpy().view(np.uint16)
        return [a[int(offs[i]) - int(offs[i0]):int(offs[i + 1]) - int(offs[i0])] for i in range(i0, i1)]

    hp, hc = host(prev), host(curr)
    shapes = [s for _, s in picked]
    per, parts, nb, _ = time_reference(names, shapes, hp, hc, args.repr, 2, 1)
    cpu = {"value": round(2 * total / statistics.mean(per) / 1e9, 4), "unit": "GB/s", "cores": 1,
           "kind": "reference", "sample": f"{len(picked)} whole tensors / {total} elements of {args.workload} "
                                           "(D2H of the benchmark's own device snapshots), reference "
                                           "encode+write+read+decode(verify=false), 1 thread",
           "parts_s": {k: round(statistics.mean(p[k] for p in parts), 4) for k in parts[0]}}

    R = reference()
    wire = R.encode_pulps(Checkpoint(1, [Tensor(n, s, a) for n, s, a in zip(names, shapes, hc)]),
                          Checkpoint(0, [Tensor(n, s, a) for n, s, a in zip(names, shapes, hp)]),
                          reprs=(args.repr,))[args.repr]
    hlen = int.from_bytes(wire[8:16], "little")
    header = json.loads(wire[16:16 + hlen])
    ref_body = wire[16 + hlen:]
    ents = {int(e["tensor"]): e for e in patch.host_entries[: patch.n_entries]}
    body = patch.body[: patch.body_bytes].cpu().numpy().tobytes()
    pos, ok, compared, changes, first = 0, True, 0, 0, True
    for h in header["tensors"]:
        t = [n for n, _ in mine].index(h["name"])
        e = ents.get(t)
        ib = ref_body[pos:pos + h["index_nbytes"]]
        vb = ref_body[pos + h["index_nbytes"]:pos + h["index_nbytes"] + h["value_nbytes"]]
        pos += h["index_nbytes"] + h["value_nbytes"]
        if e is None or int(e["count"]) != h["count"] or int(e["idx_nbytes"]) != h["index_nbytes"]:
            ok = False
            break
        di = body[int(e["idx_off"]):int(e["idx_off"]) + int(e["idx_nbytes"])]
        dv = body[int(e["val_off"]):int(e["val_off"]) + 2 * int(e["count"])]
        if args.repr == 2 and first:
            prev_changed = [k for k in ents if k < t]
            if prev_changed:
                q = max(prev_changed)
                d = (prev[int(offs[q]):int(offs[q + 1])] != curr[int(offs[q]):int(offs[q + 1])]).nonzero()
                last = int(d[-1].item())
                want0 = (int(offs[q + 1] - offs[q]) - last + int.from_bytes(ib[:4], "little")) & 0xFFFFFFFF
                ok = ok and int.from_bytes(di[:4], "little") == want0
                di, ib = di[4:], ib[4:]
        first = False
        ok = ok and di == ib and dv == vb
        compared += 1
        changes += h["count"]
    parity = {"bit_exact": bool(ok), "tensors": compared, "changes": changes,
              "reference_body_bytes": len(ref_body), "representation": REPR_NAMES[args.repr],
              "what": "reference write_patch_bytes(encode(curr, prev)) blobs of the sampled tensors vs their "
                      "sections of the device patch body, same input bytes"}
    return cpu, parity


def profiled_traffic(args, world):
    """dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch from the
    committed `ncu --set full` capture of this same configuration, else None."""
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)["k1_diff_compact"]
    except (OSError, KeyError, ValueError):
        return None
    same = (t.get("workload") == args.workload and t.get("n_gpus") == world and
            t.get("representation") == REPR_NAMES[args.repr] and abs(t.get("sparsity", -1) - args.sparsity) < 1e-9)
    return t["dram_bytes_per_launch"] if same else None


def run_e2e(args, mine, prev, curr, views, world, rank):
    """End to end through the reference-facing host API (host buffers in,
    host buffers out): paper_2602_03839_b200.host.bench_e2e."""
    from paper_2602_03839_b200 import host

    return host.bench_e2e(args, mine, prev, curr, world, rank)


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_pulse(args)


if __name__ == "__main__":
    sys.exit(main())
