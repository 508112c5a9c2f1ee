"""The paper's KV-migration microbenchmark on B200 (Fig.
"KV-Migration Latency Comparison": 0.5-5 GB of fp16 Llama-8B KV, fully
fragmented and contiguous layouts; cudaMemcpyAsync per page 0.88-9.25 s vs
Nitsum's aggregated+pipelined copy 3.6-24.8 ms on A100/H100).

One request of 4096..40960 tokens moves all 8 KV heads between two GPU slots
(a TP1 -> TP1 handoff: every byte moves). Methods:

* per-plane cudaMemcpyAsync: one call per (page, layer, K|V) plane, 4 KiB each;
  this is the "separate request for each memory page" straw-man;
* per-page cudaMemcpyAsync: one call per 256 KiB page (all layers);
* K3 + K1 (this repo): one ABI call.

Both slots live in one B200's HBM (1-GPU box), so this measures issue
overhead + HBM, not NVLink.

    python tools/kv_microbench.py --out profiles/r01_kv_microbench.jsonl
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def aggregate_pipelined(c, su, du, st, chunk_pages: int = 512):
    """The paper's mechanism built from this repo's copy
    engine: pack fragmented pages into one of two staging buffers (K2 gather),
    send the buffer with one cudaMemcpyAsync, unpack at the destination (K2
    scatter). Chunks alternate buffers; pack and send run on two streams, so
    packing chunk i+1 overlaps sending chunk i. Returns ms for all pages."""
    import ctypes

    import torch

    from paper_2605_05467_b200 import _native
    from paper_2605_05467_b200.weights import CHUNK_BYTES

    U = c.kv.unit_bytes
    dev = c.home
    stage_src = [torch.empty(chunk_pages * U, dtype=torch.uint8, device=dev) for _ in range(2)]
    stage_dst = [torch.empty(chunk_pages * U, dtype=torch.uint8, device=dev) for _ in range(2)]
    send = torch.cuda.Stream()
    p0, p1 = c.pools[0].data_ptr(), c.pools[1].data_ptr()

    def segments(pairs):
        """Upload a page-copy descriptor list once (outside the timed region)."""
        seg = np.zeros((len(pairs), 8), dtype=np.int64)
        for i, (s, d) in enumerate(pairs):
            seg[i, :6] = (s, d, 1, U, U, U)
        prefix = np.zeros(len(seg) + 1, dtype=np.int64)
        n_items = ctypes.c_int64()
        _native.call("tpr_copy_prepare", seg.ctypes.data, len(seg), CHUNK_BYTES, prefix.ctypes.data,
                     ctypes.byref(n_items))
        d = torch.from_numpy(np.concatenate([seg.reshape(-1), prefix])).to(dev)
        return d, seg.nbytes, len(seg), n_items.value

    def launch(desc, stream):
        d, off, n, items = desc
        # descriptors are reused across launches: static schedule (no claim counter)
        _native.call("tpr_weight_reshard", d.data_ptr(), d.data_ptr() + off, n, items, CHUNK_BYTES,
                     None, stream.cuda_stream)

    chunks = [(su[i:i + chunk_pages], du[i:i + chunk_pages]) for i in range(0, len(su), chunk_pages)]
    packs, unpacks = [], []
    for i, (s_units, d_units) in enumerate(chunks):
        b = i % 2
        packs.append(segments([(p0 + int(u) * U, stage_src[b].data_ptr() + k * U)
                               for k, u in enumerate(s_units)]))
        unpacks.append(segments([(stage_dst[b].data_ptr() + k * U, p1 + int(u) * U)
                                 for k, u in enumerate(d_units)]))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    packed = [torch.cuda.Event() for _ in chunks]
    sent = [torch.cuda.Event() for _ in chunks]
    e0.record(st)
    send.wait_stream(st)
    for i, (s_units, _) in enumerate(chunks):
        b = i % 2
        if i >= 2:
            st.wait_event(sent[i - 2])  # staging buffer b is free once chunk i-2 went out
        launch(packs[i], st)          # aggregate: fragmented pages -> contiguous buffer
        packed[i].record(st)
        send.wait_event(packed[i])
        nb = np.array([len(s_units) * U], np.uint64)
        src = np.array([stage_src[b].data_ptr()], np.uint64)
        dst = np.array([stage_dst[b].data_ptr()], np.uint64)
        _native.call("tpr_baseline_copy_pages", src.ctypes.data, dst.ctypes.data, nb.ctypes.data, 1, 0,
                     send.cuda_stream)  # one large send
        launch(unpacks[i], send)      # scatter into the destination's pages
        sent[i].record(send)
    st.wait_stream(send)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1)


def main():
    import torch

    from paper_2605_05467_b200 import _native, migration as M
    from paper_2605_05467_b200.geometry import LLAMA_3_1_8B
    from paper_2605_05467_b200.kvcache import PagedKvCluster

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "kv_microbench.jsonl"))
    ap.add_argument("--tokens", default="4096,8192,16384,40960")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    kv = LLAMA_3_1_8B.kv
    H = kv.total_heads
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    out = open(args.out, "w")
    for fragmented in (True, False):
        for tokens in map(int, args.tokens.split(",")):
            pages = kv.blocks(tokens)
            c = PagedKvCluster(kv, (0, 1), units_per_gpu=H * pages + 16, max_requests=1,
                               max_blocks=pages, fragmented=fragmented, seed=1)
            src = M.KvLayout((0,), 1, H, ((0, tokens),))
            dst = M.KvLayout((1,), 1, H, ((0, tokens),))
            c.admit([src], seed=3)
            fwd = M.head_transfers_array(src, dst, kv.kv_bytes_per_token_per_head)
            back = M.head_transfers_array(dst, src, kv.kv_bytes_per_token_per_head)
            nbytes = fwd.total_bytes

            def k1_time():
                ts = []
                for r in range(args.reps + 1):
                    p = fwd if r % 2 == 0 else back
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record(st)
                    c.migrate(p, validate=False)
                    e1.record(st)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1))
                if (args.reps + 1) % 2:
                    c.migrate(back, validate=False)
                return float(np.median(ts[1:]))

            k1_ms = k1_time()
            v = c.verify()
            assert v["placement_errors"] == 0 and v["word_mismatches"] == 0
            # page pairs of the last forward move (src pages on slot 0, their destination on slot 1)
            torch.cuda.synchronize()
            n_units = H * pages
            bt0 = c.block_tables[0].cpu().numpy().reshape(1, H, pages)
            ring1 = c.rings[1].cpu().numpy()
            su = bt0[0].reshape(-1).astype(np.uint64)
            head1 = c.ring_head[1]
            du = ring1[np.arange(head1, head1 + n_units) % c.units[1]].astype(np.uint64)
            p0, p1 = c.pools[0].data_ptr(), c.pools[1].data_ptr()
            U = kv.unit_bytes
            res = {"fragmented": fragmented, "tokens": tokens, "bytes": nbytes,
                   "k3_k1_ms": k1_ms}
            for name, gran, method in (("memcpy_per_plane", "plane", 0),
                                       ("memcpy_per_page", "page", 0)):
                if gran == "page":
                    s = p0 + su * U
                    d = p1 + du * U
                    b = np.full(len(s), U, np.uint64)
                else:
                    planes = np.arange(2 * kv.layers, dtype=np.uint64) * kv.plane_bytes
                    s = (p0 + su[:, None] * U + planes[None, :]).reshape(-1)
                    d = (p1 + du[:, None] * U + planes[None, :]).reshape(-1)
                    b = np.full(len(s), kv.plane_bytes, np.uint64)
                s, d, b = (np.ascontiguousarray(x, dtype=np.uint64) for x in (s, d, b))
                ts = []
                for _ in range(2):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    _native.call("tpr_baseline_copy_pages", s.ctypes.data, d.ctypes.data,
                                 b.ctypes.data, len(s), method, st.cuda_stream)
                    torch.cuda.synchronize()
                    ts.append((time.perf_counter() - t0) * 1e3)
                res[name + "_ms"] = min(ts)
                res[name + "_calls"] = int(len(s))
            res["aggregate_pipelined_ms"] = aggregate_pipelined(c, su, du, st)
            res["speedup_vs_memcpy_per_plane"] = res["memcpy_per_plane_ms"] / k1_ms
            print(json.dumps(res))
            out.write(json.dumps(res) + "\n")
            out.flush()
            del c
            torch.cuda.empty_cache()
    out.close()


if __name__ == "__main__":
    main()
