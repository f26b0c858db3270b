"""Lookahead-parallel protocol over a real 2-rank torch.distributed (gloo)
group on CPU: each rank evaluates only its shard of the step (host row plan
``shard_rows``, the mirror of the device plan), the ranks all-gather the
per-row argmax tables exactly as the device exchange does, merge, and run the
replicated step finish.  The decode must equal the single-process decode
token for token (reference SPEC.md:515,523).  The CPU oracle plays the model
(test infrastructure); the NCCL id broadcast uses the product helper."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lookahead_oracle as lo
from oracle.model_oracle import TinyTransformerOracle
from paper_2402_02057_b200.parallel import broadcast_unique_id, shard_rows

ROWS = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lp_decode(model, prompt, W, N, G, max_tokens, seed, rank, world):
    import numpy as np
    pool = lo.OraclePool(N)
    pool.seed_from_prompt(prompt)
    rng = np.random.default_rng(seed)
    window = lo.window_init(W, N, model.vocab_size, rng)
    prefix = list(prompt)
    out, steps = [], 0
    while True:
        last = prefix[-1]
        sufs = pool.lookup(last, G)
        rows = lo.build_rows(window, W, N, last, sufs)
        computed, owned = shard_rows(W, N, len(sufs), rank, world)
        # closure: every computed row's chain is computed locally
        for g in computed:
            assert set(rows.chains[g]) <= set(computed)
        table = torch.full((ROWS,), -1, dtype=torch.int32)
        am = model.argmax_rows(prefix[:-1], rows)     # (oracle evaluates all; keep owned)
        for g in owned:
            table[g] = am[g]
        gathered = [torch.empty_like(table) for _ in range(world)]
        dist.all_gather(gathered, table)
        merged = torch.stack(gathered).max(0).values.tolist()
        new_top = [merged[g] for g in rows.generators]
        acc, _ = lo.verify_greedy_rows(lambda r: merged[r], rows, sufs)
        pool.insert_all(lo.collect_ngrams(window, W, N, new_top, last))
        window = lo.window_update(window, W, N, model.vocab_size, new_top, len(acc), rng)
        prefix.extend(acc)
        steps += 1
        if lo.fold_output(out, acc, max_tokens, None):
            return out, steps


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
        raw = broadcast_unique_id(uid)
        assert raw == bytes(range(128))
        model = TinyTransformerOracle(3, 16)
        toks, steps = _lp_decode(model, [15, 9, 4, 9, 7, 8], 5, 3, 5, 24, 2, rank, world)
        results[rank] = (toks, steps)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_lp_matches_single_process():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    ref = lo.decode_lookahead(TinyTransformerOracle(3, 16), [15, 9, 4, 9, 7, 8], 5, 3, 5, 24,
                              None, 2, True)
    for r in range(world):
        toks, steps = results[r]
        assert toks == ref.tokens
        assert steps == len(ref.steps)
