"""CPU port of the per-iteration path (TEST INFRASTRUCTURE / CPU baseline only).

The reference's CPU implementation of this path is `tokensim` (pure Python,
cost-model stages: `engine.py:96-105`), so there is nothing to compile into
oracle/_ref. The measured CPU baseline is this port: the oracle scheduler
(`sched_ref.RefEngine`, pinned to the reference's golden timelines) driving an
fp32 torch-CPU decoder with dense per-request KV caches.

Bounded sample: only `sample_layers` of the model's L layers are held and run;
each step's time is scaled to the full depth as
    t_full = t_embed + (L / sample_layers) * t_layers + t_head.
Everything in the timed step is real work (no skipped tokens).
"""

from __future__ import annotations

import math
import os
import time

import numpy as np
import torch

from oracle.sched_ref import RefEngine


def _rms(x, w, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


class CpuSlice:
    def __init__(self, spec, sample_layers: int = 2, seed: int = 0, max_pos: int = 9000, threads: int | None = None):
        from oracle.model_ref import rope_table_ref as rope_table

        torch.set_num_threads(threads or os.cpu_count() or 1)
        self.threads = torch.get_num_threads()
        self.spec = spec
        self.L = sample_layers
        g = torch.Generator().manual_seed(seed)
        d, hd = spec.d_model, spec.head_dim
        sc = 1.0 / math.sqrt(2 * spec.n_layers)
        self.layers = []
        for _ in range(sample_layers):
            self.layers.append({
                "wqkv": torch.randn(spec.qkv_width, d, generator=g) * 0.02,
                "bqkv": torch.zeros(spec.qkv_width) if spec.qkv_bias else None,
                "wo": torch.randn(d, spec.n_heads * hd, generator=g) * 0.02 * sc,
                "wgu": torch.randn(2 * spec.d_ff, d, generator=g) * 0.02,
                "wd": torch.randn(d, spec.d_ff, generator=g) * 0.02 * sc,
            })
        self.embed = torch.randn(spec.vocab, d, generator=g) * 0.02
        self.lm_head = torch.randn(spec.vocab, d, generator=g) * 0.02
        self.rope = torch.from_numpy(rope_table(spec, max_pos))
        self.kv: dict[int, list] = {}
        self.tokens: dict[int, list[int]] = {}

    def _rot(self, x, pos):
        cs = self.rope[pos]
        c, s = cs[..., 0][:, None, :], cs[..., 1][:, None, :]
        h = x.shape[-1] // 2
        return torch.cat([x[..., :h] * c - x[..., h:] * s, x[..., h:] * c + x[..., :h] * s], -1)

    @torch.no_grad()
    def step(self, seqs):
        """seqs: [(rid, start, n_new, token_ids np, emits)] -> (sampled tokens, t_embed, t_layers, t_head)."""
        s = self.spec
        H, KV, hd = s.n_heads, s.n_kv_heads, s.head_dim
        t0 = time.perf_counter()
        ids = torch.from_numpy(np.concatenate([q[3] for q in seqs]).astype(np.int64))
        x = self.embed[ids]
        pos = torch.cat([torch.arange(q[1], q[1] + q[2]) for q in seqs])
        t1 = time.perf_counter()
        for li, L in enumerate(self.layers):
            h = _rms(x, 1.0, s.rms_eps)
            qkv = h @ L["wqkv"].T
            if L["bqkv"] is not None:
                qkv = qkv + L["bqkv"]
            T = x.shape[0]
            q = self._rot(qkv[:, : H * hd].view(T, H, hd), pos)
            k = self._rot(qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd), pos)
            v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
            out = torch.empty(T, H * hd)
            off = 0
            for rid, start, n, _, _ in seqs:
                cache = self.kv.setdefault(rid, [[None, None] for _ in self.layers])[li]
                if start > 0 and (cache[0] is None or cache[0].shape[0] < start):
                    # request whose earlier tokens ran before the sampled window: synthetic cache of the
                    # right length (attention cost depends on the length, not the values)
                    cache[0] = torch.randn(start, KV, hd) * 0.1
                    cache[1] = torch.randn(start, KV, hd) * 0.1
                kk = k[off:off + n] if start == 0 else torch.cat([cache[0][:start], k[off:off + n]])
                vv = v[off:off + n] if start == 0 else torch.cat([cache[1][:start], v[off:off + n]])
                cache[0], cache[1] = kk, vv
                g = H // KV
                kr, vr = kk.repeat_interleave(g, 1), vv.repeat_interleave(g, 1)
                att = torch.einsum("thd,shd->hts", q[off:off + n], kr) / math.sqrt(hd)
                qp = torch.arange(start, start + n)[:, None]
                att = att.masked_fill(torch.arange(start + n)[None, :] > qp, float("-inf")).softmax(-1)
                out[off:off + n] = torch.einsum("hts,shd->thd", att, vr).reshape(n, H * hd)
                off += n
            x = x + out @ L["wo"].T
            h = _rms(x, 1.0, s.rms_eps)
            gu = h @ L["wgu"].T
            x = x + (torch.nn.functional.silu(gu[:, : s.d_ff]) * gu[:, s.d_ff:]) @ L["wd"].T
        t2 = time.perf_counter()
        rows, off = [], 0
        for rid, start, n, _, emits in seqs:
            off += n
            if emits:
                rows.append(off - 1)
        sampled = []
        if rows:
            logits = _rms(x[rows], 1.0, s.rms_eps) @ self.lm_head.T
            sampled = logits.argmax(-1).tolist()
        t3 = time.perf_counter()
        return sampled, t1 - t0, t2 - t1, t3 - t2


def run_cpu_path(spec, requests, steps: int, warmup: int, sample_layers: int = 2, total_pages: int = 1 << 20,
                 time_budget_s: float = 120.0, threads: int | None = None, warm_decodes: int = 0,
                 warm_max_iters: int = 0):
    """Serve `requests` on the CPU port; time `steps` micro-batches after `warmup` untimed ones.

    The schedule is warmed in first WITHOUT model work (oracle scheduler only) until
    `warm_decodes` decodes run or `warm_max_iters` iterations passed, so the timed
    micro-batches have the same composition regime as the GPU bench's timed steps.
    """
    from paper_2504_14775_b200.workload import prompt_token_ids

    model = CpuSlice(spec, sample_layers, threads=threads)
    hist = {r.id: list(prompt_token_ids(r.id, r.input_tokens, spec.vocab, getattr(r, "token_seed", None)))
            for r in requests}
    per_step = []
    t_start = None
    state = {"warm": warm_decodes > 0 or warm_max_iters > 0, "it": 0}

    def forward(seq, dec, chunks, dec_stored, reqs):
        nonlocal t_start
        if state["warm"]:
            state["it"] += 1
            rd = sum(1 for r in reqs.values() if r["dec"]) + len(dec)
            if rd >= warm_decodes or state["it"] >= warm_max_iters:
                state["warm"] = False
            for rid, n in chunks:        # keep token history long enough for later decodes
                r = reqs[rid]
                if r["done"] + n >= r["target"] and r["gen"] == 0 and len(hist[rid]) <= r["done"] + n:
                    hist[rid].append(0)
            for rid in dec:
                while len(hist[rid]) <= dec_stored[rid]:
                    hist[rid].append(0)
            return
        if t_start is None:
            t_start = time.perf_counter()
        if len(per_step) >= warmup + steps or time.perf_counter() - t_start > time_budget_s:
            return
        seqs = []
        for rid in dec:
            st = dec_stored[rid] - 1
            seqs.append((rid, st, 1, np.asarray([hist[rid][st]]), True))
        for rid, n in chunks:
            r = reqs[rid]
            st = r["done"]
            emits = st + n >= r["target"] and r["gen"] == 0
            seqs.append((rid, st, n, np.asarray(hist[rid][st:st + n]), emits))
        sampled, te, tl, th = model.step(seqs)
        k = 0
        for rid, st, n, _, emits in seqs:
            if emits:
                while len(hist[rid]) <= st + n:
                    hist[rid].append(int(sampled[k]))
                k += 1
        full = te + (spec.n_layers / sample_layers) * tl + th
        per_step.append((len(sampled), sum(q[2] for q in seqs), full))

    reqs = [(r.id, r.arrival_ms, r.input_tokens, r.output_tokens) for r in requests]
    RefEngine(reqs, "throttle", 1, total_pages, 16, forward=forward).run(
        stop=lambda: len(per_step) >= warmup + steps or (
            t_start is not None and time.perf_counter() - t_start > time_budget_s))

    timed = per_step[warmup:warmup + steps]
    out_tok = sum(a for a, _, _ in timed)
    secs = sum(c for _, _, c in timed)
    return {"value": out_tok / secs if secs > 0 else 0.0, "steps": len(timed), "threads": model.threads,
            "out_tokens": out_tok, "tokens": sum(b for _, b, _ in timed), "est_full_s": secs,
            "sample": f"{sample_layers}/{spec.n_layers} layers of {spec.name} in fp32 on CPU per micro-batch, "
                      f"time scaled x{spec.n_layers / sample_layers:g} + embed + LM head; "
                      f"{len(timed)} Token-Throttling micro-batches of the bench trace"}
