"""Expert parallel on the GPU: two engines (ranks 0 and 1 of world 2), each
owning half of every layer's experts, exchange their slot buffers over CUDA
IPC peer memory inside the decode graph.  Run as two processes on cuda:0
(the single-GPU box); on an 8-GPU node the same code runs one rank per GPU.

Greedy tokens must equal the reference golden (C1 family, mixed quant), and
each rank's store event log must equal the oracle store restricted to the
rank's keys, driven by the same routing."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASE = "mq42_k2_m2"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q, case=CASE):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import json

        from oracle import engine as OE
        from oracle import model as OM
        from paper_2312_17238_b200 import CacheConfig, ExpertKey, OffloadEngine, SpeculationConfig
        from paper_2312_17238_b200.expert_parallel import connect
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        with open(os.path.join(root, "tests", "golden", "engine_cases.json")) as fh:
            meta = json.load(fh)
        cfg = OM.ModelConfig(**meta["config"])
        name, qb, k, b, m, ntok = next(c for c in meta["cases"] if c[0] == case)
        if qb:
            fq, pay, attn = OE.build_mixed_quant(OM.init_params(cfg), cfg, *qb)
            pay = {ExpertKey(*kk): v for kk, v in pay.items()}
        else:  # fp32 experts: CUDA-core GEMV layout, exchange by k_exchange
            fq, pay, attn = OM.init_params(cfg), None, None
        eng = OffloadEngine(OM.Model(cfg, fq), CacheConfig(k, b),
                            SpeculationConfig(enabled=m > 0, m=max(m, 1)),
                            payloads=pay, record_hidden=True, attn_blocks=attn, device=0,
                            ep_rank=rank, ep_world=world)
        connect(eng)
        data = np.load(os.path.join(root, "tests", "golden", "engine_golden.npz"))
        eng.prefill([int(t) for t in data["prompt"]])
        res = eng.decode(ntok)
        ev = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved)
              for e in eng.events]
        recs = [(r.token_pos, r.layer, tuple(r.experts), r.hidden) for r in res.trace.records]
        q.put((rank, res.tokens, res.final_logits, ev, recs, None))
        eng.close()
    except Exception as ex:  # surface the failure to the parent
        import traceback
        q.put((rank, None, None, None, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case", [CASE, "fp32_k2_m2"])
def test_ep_world2_matches_reference(case):
    """mq42 (tensor-core layout): the exchange fused into the down GEMV;
    fp32 experts (CUDA-core layout): the separate k_exchange kernel."""
    import torch.multiprocessing as mp

    from oracle import engine as OE
    from oracle import model as OM
    from oracle.store import CacheConfig, ExpertStore
    from paper_2312_17238_b200.expert_parallel import owned_keys
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, case)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=540) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
    for o in outs:
        assert o[5] is None, o[5]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    data = np.load(os.path.join(root, "tests", "golden", "engine_golden.npz"))
    import json
    with open(os.path.join(root, "tests", "golden", "engine_cases.json")) as fh:
        meta = json.load(fh)
    cfg = OM.ModelConfig(**meta["config"])
    name, qb, k, b, m, ntok = next(c for c in meta["cases"] if c[0] == case)
    gold = [int(t) for t in data[f"{case}/tokens"]]
    for rank, toks, logits, ev, recs, _ in outs:
        assert toks == gold
        ref = data[f"{case}/final_logits"].astype(np.float64)
        assert np.abs(logits - ref).max() <= 2e-3 * np.abs(ref).max() + 1e-4
    # both ranks saw identical routing and hidden states (replicated dense path)
    r0, r1 = outs[0][4], outs[1][4]
    assert [x[:3] for x in r0] == [x[:3] for x in r1]
    # each rank's events == oracle store on its keys, driven by that routing
    L, E = cfg.n_layers, cfg.n_experts
    plen = len(data["prompt"])
    if qb:
        fq, pay, _ = OE.build_mixed_quant(OM.init_params(cfg), cfg, *qb)
        ebytes = OE.payload_bytes(pay[(0, 0)])
    else:
        fq = OM.init_params(cfg)
        ebytes = OE.payload_bytes(OM.Model(cfg, fq).expert(0, 0))
    gates = [fq[f"layers.{l}.gate"] for l in range(L)]
    for rank, toks, logits, ev, recs, _ in outs:
        own = owned_keys(L, E, rank, 2)
        st = ExpertStore(L, E, CacheConfig(k, b, ebytes), owned=own)
        by_tok = {}
        for t, l, ex, h in recs:
            by_tok.setdefault(t, {})[l] = (ex, h)
        for l in range(L):  # prefill: first-use order, no speculation
            seen = set()
            for t in range(plen):
                for e in by_tok[t][l][0]:
                    if e not in seen:
                        seen.add(e)
                        if (l, e) in own:
                            st.acquire(l, e, t)
        for t in sorted(x for x in by_tok if x >= plen):
            for l in range(L):
                ex, h = by_tok[t][l]
                for e in ex:
                    if (l, e) in own:
                        st.acquire(l, e, t)
                if m > 0 and l + 1 < L:
                    g = OM.top_k(h @ gates[l + 1], m)
                    keys = [(l + 1, int(x)) for x in g if (l + 1, int(x)) in own]
                    if keys:
                        st.speculative_load(keys, t, current_layer=l)
        assert ev == st.events, f"rank {rank}"


@pytest.mark.timeout(300)
def test_nccl_transport_world1_matches_reference():
    """The NCCL transport (moe_ep_connect_nccl: one ncclAllGather per layer and
    position, captured in the decode graph, rank-major combine) on a one-rank
    communicator -- the only NCCL shape one GPU can run.  Tokens equal the
    reference golden, the event log equals the single-GPU engine's, logits
    within the parity tolerance."""
    import json

    from oracle import engine as OE
    from oracle import model as OM
    from paper_2312_17238_b200 import CacheConfig, ExpertKey, OffloadEngine, SpeculationConfig
    from paper_2312_17238_b200.expert_parallel import nccl_unique_id
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "tests", "golden", "engine_cases.json")) as fh:
        meta = json.load(fh)
    cfg = OM.ModelConfig(**meta["config"])
    name, qb, k, b, m, ntok = next(c for c in meta["cases"] if c[0] == CASE)
    fq, pay, attn = OE.build_mixed_quant(OM.init_params(cfg), cfg, *qb)
    data = np.load(os.path.join(root, "tests", "golden", "engine_golden.npz"))
    prompt = [int(t) for t in data["prompt"]]
    out = []
    for nccl in (False, True):
        eng = OffloadEngine(OM.Model(cfg, fq), CacheConfig(k, b),
                            SpeculationConfig(enabled=m > 0, m=max(m, 1)),
                            payloads={ExpertKey(*kk): v for kk, v in pay.items()},
                            record_hidden=False, attn_blocks=attn, device=0)
        if nccl:
            eng.ep_connect_nccl(nccl_unique_id())
        eng.prefill(prompt)
        res = eng.decode(ntok)
        ev = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved)
              for e in eng.events]
        out.append((res.tokens, res.final_logits, ev))
        eng.close()
    gold = [int(t) for t in data[f"{CASE}/tokens"]]
    ref = data[f"{CASE}/final_logits"].astype(np.float64)
    (t0, l0, e0), (t1, l1, e1) = out
    assert t0 == gold and t1 == gold
    assert e1 == e0
    assert np.abs(l1 - ref).max() <= 2e-3 * np.abs(ref).max() + 1e-4
