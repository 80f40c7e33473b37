"""Decode benchmark of the B200 MoE offloading engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], "C2"): Mixtral-8x7B-shaped model
(V=32000, d=4096, L=32, H=32, f=14336, E=8, top-2), random-init synthetic
weights (counter hash, oracle/model.py synth_params) quantized on device with
the reference quantizer: 4-bit attention, 3-bit experts, fp16 embeddings /
lm_head / gates.  LRU cache k=4 experts per layer, b=4 staging buffers, no
prefetch; experts live in a pinned host arena and miss loads stream over
PCIe.  A "step" is one greedy decode token after a 16-token prompt.

One JSON line on rank 0.  ``value`` = tokens/s from CUDA events on the
engine's compute stream around K device-greedy decode steps; ``e2e`` = the same
through the public API with a host sampler (per step: H2D token, D2H logits).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s Mixtral-8x7B-shape @cache k=2/4; expert hit rate; H2D GB/s"
MIXTRAL = dict(vocab_size=32000, d_model=4096, n_layers=32, n_heads=32, d_ffn=14336,
               n_experts=8, top_k_gate=2, seed=0, max_seq_len=256)
CONFIGS = {  # name -> (attn_bits, expert_bits, k, spec m)
    "c2": (4, 3, 4, 0),
    "c3": (4, 2, 2, 2),
}
PRESET = {2: (16, 128), 3: (64, 128), 4: (64, 256)}


def matrix_payload_bytes(K, N, bits):
    """quant.payload_nbytes of a K x N block (quant.py:332-343)."""
    g, sg = PRESET[bits]
    ng = K * N // g
    return K * N * bits // 8 + ng + 2 * (-(-ng // (sg // g))) + 4 * (-(-ng // sg))


def expert_bytes(cfg, bits):
    d, f = cfg["d_model"], cfg["d_ffn"]
    return 2 * matrix_payload_bytes(d, f, bits) + matrix_payload_bytes(f, d, bits)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cfg_obj(d):
    from oracle.model import ModelConfig  # plain dataclass, no oracle logic involved
    return ModelConfig(**d)


def build_engine(cfg, cname, seed, device=0, rank=0, world=1):
    """World > 1: expert parallel, this rank owns 1/world of every layer's
    experts with LRU capacity ceil(k/world) (capped budget per GPU, C4)."""
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    from paper_2312_17238_b200 import synthetic_model
    from paper_2312_17238_b200.expert_parallel import connect, local_cache_k
    ab, xb, k, m = CONFIGS[cname]
    cobj = cfg_obj(cfg)
    kl = local_cache_k(k, cfg["n_experts"], world) if world > 1 else k
    eng = OffloadEngine(synthetic_model(cobj, seed), CacheConfig(k=kl, b=4),
                        SpeculationConfig(enabled=m > 0, m=max(m, 1)), record_hidden=False,
                        synth=(seed, ab, xb), expert_bytes=expert_bytes(cfg, xb), device=device,
                        ep_rank=rank, ep_world=world)
    if world > 1:
        connect(eng)
    return eng


def window_stats(events, cfg, xb):
    from paper_2312_17238_b200 import recall
    miss = sum(1 for e in events if e.kind == "miss_load")
    spec = sum(1 for e in events if e.kind == "speculative_load")
    shit = sum(1 for e in events if e.kind == "staging_hit")
    moved = sum(e.bytes_moved for e in events if e.kind in ("miss_load", "speculative_load"))
    eb = max((e.bytes_moved for e in events), default=0)
    return {"hit_rate": recall(events) if events else None,
            "hit_rate_device_only": recall(events, "device_only") if events else None,
            "miss_loads": miss, "speculative_loads": spec, "staging_hits": shit,
            "h2d_bytes": moved,
            # bytes any engine must move for these decisions: every miss, and
            # the speculative copy behind every staging hit
            "h2d_bytes_needed": (miss + shit) * eb}


def _progress(msg):
    if os.environ.get("MOE_BENCH_VERBOSE"):
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_b200(args, rank, world):
    import ctypes as C

    from paper_2312_17238_b200 import _lib
    cfg = dict(MIXTRAL)
    ab, xb, k, m = CONFIGS[args.config]
    t_build = time.perf_counter()
    eng = build_engine(cfg, args.config, args.seed, device=args.device, rank=rank, world=world)
    t_build = time.perf_counter() - t_build
    _progress(f"engine built in {t_build:.1f}s")
    V = cfg["vocab_size"]
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, V, 16)]
    eng.prefill(prompt)
    _progress("prefill done")
    eng.decode(args.warmup)
    _progress("warmup done")
    n0 = len(eng.events)
    s0 = eng.stats()
    L = _lib.lib()
    ncu_range = os.environ.get("MOE_NCU_RANGE") == "1"  # ncu --profile-from-start off
    with ClockSampler(args.device) as clk:
        if ncu_range:
            _lib.check(L.moe_profiler_range(1))
        res = eng.decode(args.steps)
        if ncu_range:
            _lib.check(L.moe_profiler_range(0))
    s1 = eng.stats()
    ms_tot = s1["last_call_ms"]
    launches = s1["kernel_launches"]
    ev = eng.events[n0:]
    win = window_stats(ev, cfg, xb)
    time.sleep(0.5)  # let in-flight speculative copies land before reading copy stats
    s1 = eng.stats()
    tok_s = args.steps / (ms_tot / 1e3)

    # ---- per-kernel CUDA-event timing pass (separate from the headline: the
    # events between launches disable programmatic dependent launch overlap)
    kp = max(1, min(8, args.steps))
    eng.prefill(prompt)
    _lib.check(L.moe_set_profiling(eng._h, 1))
    eng.decode(kp)
    kms = (C.c_double * 5)()
    kcnt = (C.c_int64 * 5)()
    _lib.check(L.moe_kernel_times(eng._h, kms, kcnt))
    _lib.check(L.moe_set_profiling(eng._h, 0))
    prof_ms_step = eng.stats()["last_call_ms"] / kp

    # ---- device timeline of one token (%globaltimer spans per kernel, PDL on)
    timeline = None
    try:
        eng.prefill(prompt)
        eng.decode(2)
        _lib.check(L.moe_timeline(eng._h, 1))
        eng.decode(1)
        n = C.c_int32()
        _lib.check(L.moe_read_timeline(eng._h, None, 0, C.byref(n)))
        buf = (C.c_uint64 * (10 * n.value))()
        _lib.check(L.moe_read_timeline(eng._h, buf, 5 * n.value, C.byref(n)))
        _lib.check(L.moe_timeline(eng._h, 0))
        raw = np.array(buf[:], dtype=np.float64)
        st = raw[0:2 * n.value:2]
        en = raw[1:2 * n.value:2]
        marks = raw[2 * n.value:].reshape(n.value, 8)
        ok = (en > 0) & (st < 2 ** 63)
        t0 = st[ok].min()
        names = ["qkv", "attention", "wo", "tail", "expert_up", "expert_down", "combine_ln"]
        nl = cfg["n_layers"]
        kinds = {}
        for i, nm in enumerate(names):
            idx = [1 + 8 * l + i for l in range(nl)]
            d = [(en[j] - st[j]) / 1e3 for j in idx if ok[j]]
            if d:
                kinds[nm] = {"avg_us": round(float(np.mean(d)), 2),
                             "median_us": round(float(np.median(d)), 2),
                             "sum_us": round(float(np.sum(d)), 1)}
        for nm, j in (("embed", 0), ("lm_head", 1 + 8 * nl), ("logits", 2 + 8 * nl)):
            if ok[j]:
                kinds[nm] = {"avg_us": round((en[j] - st[j]) / 1e3, 2),
                             "sum_us": round((en[j] - st[j]) / 1e3, 1)}
        phases = {}
        for nm, kind, nph in (("tail", 3, 8), ("combine_ln", 6, 3), ("attention", 1, 3),
                              ("qkv", 0, 5), ("wo", 2, 5), ("expert_up", 4, 5),
                              ("expert_down", 5, 5)):
            rows = [marks[1 + 8 * l + kind] for l in range(nl) if ok[1 + 8 * l + kind]]
            starts = [st[1 + 8 * l + kind] for l in range(nl) if ok[1 + 8 * l + kind]]
            if rows:
                mk = np.array(rows)[:, :nph]
                prev = np.concatenate([np.array(starts)[:, None], mk[:, :-1]], axis=1)
                phases[nm] = [round(float(x), 2) for x in ((mk - prev) / 1e3).mean(axis=0)]
        # GEMV block 0: release delay after the earliest CTA, then its own prologue
        for nm, kind in (("qkv", 0), ("wo", 2), ("expert_up", 4), ("expert_down", 5)):
            rows = [(marks[1 + 8 * l + kind][5] - st[1 + 8 * l + kind],
                     marks[1 + 8 * l + kind][0] - marks[1 + 8 * l + kind][5])
                    for l in range(nl) if ok[1 + 8 * l + kind] and marks[1 + 8 * l + kind][5] > 0]
            if rows:
                r = np.array(rows) / 1e3
                phases[nm + "_blk0"] = [round(float(r[:, 0].mean()), 2),
                                        round(float(r[:, 1].mean()), 2)]
            # epilogue split: warp skew (loop done -> all warps), smem stores, sums + adds
            ep = [(marks[1 + 8 * l + kind][6] - marks[1 + 8 * l + kind][3],
                   marks[1 + 8 * l + kind][7] - marks[1 + 8 * l + kind][6],
                   marks[1 + 8 * l + kind][4] - marks[1 + 8 * l + kind][7])
                  for l in range(nl) if ok[1 + 8 * l + kind] and marks[1 + 8 * l + kind][7] > 0]
            if ep:
                phases[nm + "_epilogue"] = [round(float(x), 2) for x in np.array(ep).mean(0) / 1e3]
        # QKV with the fused combine: residual loads, LN statistics, own rows
        cm = [(marks[1 + 8 * l][6] - marks[1 + 8 * l][5], marks[1 + 8 * l][7] - marks[1 + 8 * l][6],
               marks[1 + 8 * l][0] - marks[1 + 8 * l][7])
              for l in range(1, nl) if ok[1 + 8 * l] and marks[1 + 8 * l][7] > marks[1 + 8 * l][6] > 0]
        if cm:
            phases["qkv_combine"] = [round(float(x), 2) for x in np.array(cm).mean(0) / 1e3]
        # tail thread-0 sub-phases (marks in the layer's exchange slot on one GPU)
        if world == 1:
            sub = [(marks[1 + 8 * l + 7][:2] - marks[1 + 8 * l + 3][5]) / 1e3 for l in range(nl)
                   if ok[1 + 8 * l + 3] and marks[1 + 8 * l + 7][1] > 0]
            if sub:
                sub = np.array(sub)
                phases["tail_thread0"] = [round(float(sub[:, 0].mean()), 2),
                                          round(float((sub[:, 1] - sub[:, 0]).mean()), 2)]
        span = (en[ok].max() - t0) / 1e3
        timeline = {"token_span_us": round(float(span), 1),
                    "busy_sum_us": round(float(sum(v["sum_us"] for v in kinds.values())), 1),
                    "kernels": kinds, "phases_us": phases,
                    "how": "one decode token after the timed region, graph + PDL; per kernel "
                           "earliest CTA start (after griddepcontrol.wait) to latest CTA end, "
                           "%globaltimer"}
    except Exception as ex:  # profiling aid only
        timeline = {"error": str(ex)}

    # ---- e2e through the public API: host sampler, per-step H2D token + D2H logits
    e2e = None
    if not args.no_e2e:
        def host_greedy(logits):
            return int(np.argmax(logits))
        ke = min(args.steps, cfg["max_seq_len"] - 16 - args.warmup)
        eng.prefill(prompt)
        eng.decode(args.warmup, sampler=host_greedy)  # same warm cache as the timed run
        t0 = time.perf_counter()
        eng.decode(ke, sampler=host_greedy)
        dt = time.perf_counter() - t0
        e2e = {"value": round(ke / dt, 3), "unit": "tokens/s", "h2d_bytes_per_step": 4,
               "d2h_bytes_per_step": 4 * V, "steps": ke,
               "api": "OffloadEngine.decode(sampler=host callable) -> moe_step per token",
               "h2d_expert_bytes_per_step": None}

    # ---- roofline of the dominant kernel (expert up-projection GEMV, hit path)
    peaks, peak_kind = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    up_bytes = 2 * cfg["n_experts"] // cfg["n_experts"] * 2 * matrix_payload_bytes(
        cfg["d_model"], cfg["d_ffn"], xb)
    dn_bytes = 2 * matrix_payload_bytes(cfg["d_ffn"], cfg["d_model"], xb)
    avg = lambda i: kms[i] / max(kcnt[i], 1)  # noqa: E731
    up_gbs = up_bytes / (avg(2) * 1e-3) / 1e9 if kcnt[2] else None
    dn_gbs = dn_bytes / (avg(3) * 1e-3) / 1e9 if kcnt[3] else None
    attn_block = matrix_payload_bytes(cfg["d_model"], cfg["d_model"], ab)
    qkv_gbs = 3 * attn_block / (avg(0) * 1e-3) / 1e9 if kcnt[0] else None
    lm_gbs = cfg["d_model"] * V * 2 / (avg(4) * 1e-3) / 1e9 if kcnt[4] else None
    prof_path = os.path.join(ROOT, "profiles", "ncu_expert_up.json")
    traffic = None
    if os.path.exists(prof_path):
        with open(prof_path) as fh:
            prof = json.load(fh)
        if f"k_gemv<{xb}>" in prof.get("kernel", ""):  # the capture is of this config's kernel
            traffic = prof.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": f"k_gemv<{xb}> expert up-projection (W1+W3 of 2 experts)",
                "achieved": round(up_gbs, 1) if up_gbs else None, "peak": hbm, "unit": "GB/s",
                "frac": round(up_gbs / hbm, 4) if up_gbs else None, "traffic": traffic,
                "algorithmic_bytes_per_launch": up_bytes,
                "avg_launch_us": round(avg(2) * 1e3, 2), "peak_kind": peak_kind,
                "timing": f"CUDA events around each launch on the compute stream over a {kp}-token "
                          f"pass after the timed region ({prof_ms_step:.3f} ms/token with events)",
                "others_gbs": {"expert_down": dn_gbs and round(dn_gbs, 1),
                               "attn_qkv": qkv_gbs and round(qkv_gbs, 1),
                               "lm_head": lm_gbs and round(lm_gbs, 1)}}
    # north-star end-to-end roofline: max(hit bytes / HBM, miss bytes / H2D)
    hit_bytes_tok = (cfg["n_layers"] * (4 * attn_block + 2 * cfg["d_model"] * cfg["n_experts"]
                                        + 2 * expert_bytes(cfg, xb)) + cfg["d_model"] * V * 2)
    miss_bytes_tok = win["h2d_bytes_needed"] / args.steps
    logical_bytes_tok = win["h2d_bytes"] / args.steps
    copies = s1["h2d_copies"] - s0["h2d_copies"]
    cbytes = s1["h2d_bytes"] - s0["h2d_bytes"]
    cbusy = s1["h2d_busy_ms"] - s0["h2d_busy_ms"]
    h2d_gbs = cbytes / (cbusy * 1e-3) / 1e9 if cbusy > 0 else None
    h2d_peak = float(peaks.get("h2d_gbs", 55.4))
    t_floor = max(hit_bytes_tok / (hbm * 1e9), miss_bytes_tok / (h2d_peak * 1e9))
    rl_e2e = {"hit_bytes_per_token": hit_bytes_tok, "miss_bytes_per_token": miss_bytes_tok,
              "miss_bytes_def": "(MISS_LOAD + STAGING_HIT) x expert_bytes: the copies the "
                                "reference's decisions require",
              "event_log_load_bytes_per_token": logical_bytes_tok,
              "physical_h2d_bytes_per_token": round(cbytes / args.steps),
              "hbm_floor_ms": round(hit_bytes_tok / (hbm * 1e9) * 1e3, 4),
              "h2d_floor_ms": round(miss_bytes_tok / (h2d_peak * 1e9) * 1e3, 4),
              "h2d_peak_gbs": h2d_peak, "frac": round(t_floor / (ms_tot / 1e3 / args.steps), 4),
              "bound": "h2d" if miss_bytes_tok / h2d_peak > hit_bytes_tok / hbm else "hbm"}
    if e2e is not None:
        e2e["h2d_expert_bytes_per_step"] = int(miss_bytes_tok)
    # the same kernel from the device timeline (graph + PDL, as in the timed run):
    # median span over the token's layers, i.e. the hit-path launches
    try:
        up_med = timeline["kernels"]["expert_up"]["median_us"]
        roofline["timeline_median_us"] = up_med
        roofline["achieved_timeline"] = round(up_bytes / (up_med * 1e-6) / 1e9, 1)
        roofline["frac_timeline"] = round(up_bytes / (up_med * 1e-6) / 1e9 / hbm, 4)
    except (KeyError, TypeError):
        pass
    line = {
        "metric": METRIC, "value": round(tok_s, 3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_tot / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: random-init counter-hash weights quantized on device; prompt = "
                "default_rng(0).integers(0, 32000, 16)",
        "config": {"workload": f"{args.config.upper()}: Mixtral-8x7B-shape "
                               f"{ab}-bit attn / {xb}-bit experts, LRU k={k}, b=4, "
                               f"prefetch m={m}, greedy decode",
                   "model": "mixtral-8x7b-shape", "global_batch": 1, "seq_len": 16 + args.warmup,
                   "parallelism": f"ep{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (5.9 GB of weights read per token)",
                   "expert_bytes": expert_bytes(cfg, xb)},
        "hit_rate": win["hit_rate"], "hit_rate_device_only": win["hit_rate_device_only"],
        "h2d_gbs": round(h2d_gbs, 2) if h2d_gbs else None,
        "h2d_gbs_wall": round(win["h2d_bytes"] / (ms_tot / 1e3) / 1e9, 2),
        "miss_loads_per_token": win["miss_loads"] / args.steps,
        "spec_loads_per_token": win["speculative_loads"] / args.steps,
        "roofline": roofline, "roofline_e2e": rl_e2e, "e2e": e2e, "timeline": timeline,
        "gpu_launches": launches, "gpu_launches_per_step": round(launches / args.steps, 1),
        "clocks": clk.summary(), "build_s": round(t_build, 1),
        "tokens": res.tokens[:8],
    }
    eng.close()
    return line


def device_helpers():
    import ctypes as C

    from oracle import model as OM
    from oracle import quant as OQ
    from paper_2312_17238_b200 import _lib
    L = _lib.lib()

    def dsynth(tid, shape, std):
        n = int(np.prod(shape))
        out = np.empty(n, np.float32)
        _lib.check(L.moe_synth_tensor_device(0, tid, n, float(OM.synth_scale(std)),
                                             out.ctypes.data_as(_lib.FP)))
        return out.reshape(shape)

    def dquant(w, bits):
        sch = OQ.PRESETS[bits]
        K, N = w.shape
        ng = K * N // sch.group_size
        nr = -(-ng // sch.scale_group_size)
        nsg = -(-ng // (sch.scale_group_size // sch.group_size))
        codes = np.empty(K * N * bits // 8, np.uint8)
        zeros = np.empty(ng, np.uint8)
        zs, zo, sc = np.empty(nr, np.uint16), np.empty(nr, np.uint16), np.empty(nsg, np.uint16)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        w = np.ascontiguousarray(w, np.float32)
        _lib.check(L.moe_quantize_device(w.ctypes.data_as(_lib.FP), K, N, bits, sch.group_size,
                                         sch.scale_group_size, vp(codes), vp(zeros), vp(zs),
                                         vp(zo), vp(sc)))
        return OQ.QuantizedBlock(sch, codes.tobytes(), zeros, zs.view(np.float16),
                                 zo.view(np.float16), sc.view(np.float16), (K, N), 0)
    return dquant, dsynth


def cpu_reference(args, steps, sample_layers=2):
    """Oracle port of the reference path on the host cores (bounded sample)."""
    from oracle import cpu_bench
    ab, xb, k, _ = CONFIGS[args.config]
    dquant, dsynth = device_helpers()
    model, payloads = cpu_bench.build_sample(dquant, dsynth, cfg_obj(MIXTRAL), args.seed, ab, xb,
                                             n_layers_sample=sample_layers)
    times, threads = cpu_bench.time_steps(model, payloads, steps, k=k)
    return times, threads


def main():
    if os.environ.get("MOE_FAULTHANDLER"):
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["MOE_FAULTHANDLER"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=list(CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--k", type=int, default=None, help="sweep: override the LRU cache size")
    ap.add_argument("--m", type=int, default=None, help="sweep: override the prefetch depth")
    args = ap.parse_args()
    if args.k is not None or args.m is not None:  # C5 sweep point derived from --config
        ab, xb, k, m = CONFIGS[args.config]
        k = k if args.k is None else args.k
        m = m if args.m is None else args.m
        name = f"{args.config}_k{k}_m{m}"
        CONFIGS[name] = (ab, xb, k, m)
        args.config = name
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    args.device = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("MOE_BENCH_DEVICE") is not None:  # test aid: all ranks on one GPU
        args.device = int(os.environ["MOE_BENCH_DEVICE"])

    if args.impl == "reference":
        if rank != 0:
            return
        times, threads = cpu_reference(args, args.warmup + args.steps)
        t = times[args.warmup:]
        v = len(t) / sum(t)
        line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "tokens/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(1e3 * sum(t) / len(t), 1), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (same weights as the b200 arm)",
                "config": {"workload": f"{args.config.upper()} (see b200 arm)",
                           "model": "mixtral-8x7b-shape"},
                "cpu_baseline": {"value": round(v, 6), "unit": "tokens/s", "cores": threads,
                                 "kind": "port",
                                 "sample": "each step: 1 greedy token through 2 of 32 Mixtral-"
                                           "width layers (dequantize-on-acquire, numpy), "
                                           "extrapolated to 32 layers + lm_head"},
                "e2e": {"value": round(v, 6), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    line = run_b200(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([line["ms_per_step"]], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        line["ms_per_step"] = float(t.item())
        # one batch-1 sequence decoded by `world` expert-parallel ranks: the
        # job's throughput is that sequence's tokens/s (slowest rank's clock)
        line["value"] = round(1e3 / line["ms_per_step"], 3)
        line["scaling"] = "strong"
        line["config"]["parallelism"] = f"ep{world}"
        if line.get("e2e"):
            e = torch.tensor([line["e2e"]["value"]], dtype=torch.float64)
            dist.all_reduce(e, op=dist.ReduceOp.MIN)
            line["e2e"]["value"] = float(e.item())
        dist.barrier()
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        times, threads = cpu_reference(args, args.cpu_steps)
        v = len(times) / sum(times)
        line["cpu_baseline"] = {"value": round(v, 6), "unit": "tokens/s", "cores": threads,
                                "kind": "port",
                                "sample": f"{args.cpu_steps} greedy tokens through 2 of 32 "
                                          "Mixtral-width layers (numpy oracle, "
                                          "dequantize-on-acquire), extrapolated to 32 layers"}
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
