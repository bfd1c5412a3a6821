"""GPU tests of the executed recovery path: K5 backup gather to pinned host,
K6 restore scatter, and the plan-driven restore of a failed rank's KV onto a
survivor (bit-exact)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cache(owner, rank, routing, lens, order="shuffled", seed=0):
    from paper_2511_14116_b200.kvcache import PagedKVCache, RankWork
    work = RankWork.build(np.asarray(owner, dtype=np.int32), rank, routing, len(lens))
    cache = PagedKVCache(work, max(lens), 4, page_order=order, seed=seed)
    cache.set_lengths(lens)
    return work, cache


def _fill(cache, work, lens, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    seqs = np.concatenate([np.full(lens[work.item_req[i]], i) for i in range(work.n_items)])
    poss = np.concatenate([np.arange(lens[work.item_req[i]]) for i in range(work.n_items)])
    k = torch.randn((len(seqs), 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((len(seqs), 128), device="cuda", generator=g).to(torch.bfloat16)
    cache.write_tokens(seqs, poss, k, v)
    return seqs, poss, k, v


def test_backup_then_restore_is_bitexact():
    from paper_2511_14116_b200.recovery_exec import KVBackupExecutor, restore_pages
    from oracle.placement import owner_table
    lens = [64, 48, 16, 80]
    owner = owner_table("hybrid", 2, 8, range(3))
    work, cache = _cache(owner, 0, {r: r % 3 for r in range(4)}, lens)
    seqs, poss, k, v = _fill(cache, work, lens, 1)
    bk = KVBackupExecutor(cache)
    n1 = bk.sync({r: lens[r] // 2 for r in range(4)})      # half the context first
    n2 = bk.sync({r: lens[r] for r in range(4)})           # then the rest
    bk.wait()
    assert n1 > 0 and n2 > 0
    assert bk.bytes_copied == (n1 + n2) * 8192
    for r in range(4):
        assert bk.backed_tokens(r) == lens[r] // 16 * 16
    used = np.concatenate([cache.block_table[i, :(lens[work.item_req[i]] + 15) // 16].cpu().numpy()
                           for i in range(work.n_items)])
    cache.pool.zero_()                                     # lose the GPU copy
    restore_pages(cache.pool, used, bk.host, used)
    torch.cuda.synchronize()
    k2, v2 = cache.read_tokens(seqs, poss)
    assert torch.equal(k, k2) and torch.equal(v, v2)


def test_page_aligned_watermark_and_incremental():
    from paper_2511_14116_b200.recovery_exec import KVBackupExecutor
    owner = np.zeros((1, 1), dtype=np.int32)
    work, cache = _cache(owner, 0, {0: 0, 1: 0}, [40, 40])
    bk = KVBackupExecutor(cache)
    assert len(bk.pending_pages({0: 15, 1: 40})) == 2      # req1: 2 full pages
    assert len(bk.pending_pages({0: 16, 1: 40})) == 1      # req0 page 0 completes
    assert len(bk.pending_pages({0: 16, 1: 40})) == 0      # nothing new
    assert bk.backed_tokens(0) == 16 and bk.backed_tokens(1) == 32


def test_restore_failed_rank_onto_survivor_per_plan():
    """hybrid(4) rank 3 fails; on-demand target makes its heads replicated;
    the survivor's new DP items for routed requests get their pages from
    rank 3's host backup (the pcie_host kv_slice transfers of
    plan_kv_recovery) and then decode exactly like before the failure."""
    import math
    from paper_2511_14116_b200.core import ModelSpec
    from paper_2511_14116_b200.kvcache import RankWork
    from paper_2511_14116_b200.placement import make_placement, owner_array
    from paper_2511_14116_b200.recovery import (BackupState, plan_kv_recovery,
                                                plan_weight_recovery)
    from paper_2511_14116_b200.recovery_exec import KVBackupExecutor, restore_pages
    m = ModelSpec(num_layers=2, num_kv_heads=4, num_q_heads=16, head_dim=128, hidden_dim=512,
                  ffn_intermediate_dim=1024)
    B, lens = 6, [33, 64, 17, 48, 5, 40]
    old = make_placement("hybrid", m, range(4))
    routing = {r: r % 4 for r in range(B)}
    w3, c3 = _cache(owner_array(old, 4), 3, routing, lens, seed=3)
    _fill(c3, w3, lens, 7)
    bk = KVBackupExecutor(c3)
    bk.sync({r: lens[r] for r in range(B)})
    bk.wait()
    rp = plan_weight_recovery(m, old, [0, 1, 2], "on_demand")
    new = rp.target_plan("hybrid", m)
    new_routing = {r: r % 3 for r in range(B)}
    backup = BackupState(host_memory_bytes=10 ** 12, kv_bytes_per_token=m.kv_bytes_per_token())
    for r in range(B):
        backup.register(r)
        backup.backed[r] = bk.backed_tokens(r)
    kp = plan_kv_recovery(backup, old, new, m, {r: lens[r] for r in range(B)}, routing,
                          new_routing, "host_restore")
    for g in (0, 1, 2):
        wg, cg = _cache(owner_array(new, 4), g, new_routing, lens, seed=10 + g)
        ids, slots = [], []
        for t in kp.transfers:
            if t.medium != "pcie_host" or t.dest_gpu != g:
                continue
            r, layer, head = t.detail
            tokens = t.num_bytes // m.kv_bytes_per_head_token()
            old_i = [i for i in range(w3.n_items) if w3.item_req[i] == r and w3.item_head[i] == head
                     and w3.seg_items[layer] <= i < w3.seg_items[layer + 1]][0]
            new_i = [i for i in range(wg.n_items) if wg.item_req[i] == r and wg.item_head[i] == head
                     and wg.seg_items[layer] <= i < wg.seg_items[layer + 1]][0]
            npg = math.ceil(tokens / 16)
            slots.extend(c3.block_table[old_i, :npg].tolist())
            ids.extend(cg.block_table[new_i, :npg].tolist())
            # read both sides
        if not ids:
            continue
        restore_pages(cg.pool, ids, bk.host, slots)
        torch.cuda.synchronize()
        for t in kp.transfers:
            if t.medium != "pcie_host" or t.dest_gpu != g:
                continue
            r, layer, head = t.detail
            tokens = t.num_bytes // m.kv_bytes_per_head_token()
            old_i = [i for i in range(w3.n_items) if w3.item_req[i] == r and w3.item_head[i] == head
                     and w3.seg_items[layer] <= i < w3.seg_items[layer + 1]][0]
            new_i = [i for i in range(wg.n_items) if wg.item_req[i] == r and wg.item_head[i] == head
                     and wg.seg_items[layer] <= i < wg.seg_items[layer + 1]][0]
            pos = np.arange(tokens)
            ko, vo = c3.read_tokens(np.full(tokens, old_i), pos)
            kn, vn = cg.read_tokens(np.full(tokens, new_i), pos)
            assert torch.equal(ko, kn) and torch.equal(vo, vn)
