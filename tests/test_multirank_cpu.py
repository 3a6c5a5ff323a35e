"""The N > 1 path on CPU (world size 2 and 3, gloo): row-block sharding
 with the library's own shard slicing (cdn_debug_host_walk_shard
cuts the streams and rebases row_ptr exactly as cdn_model_load_layer does), the
bootstrap-blob broadcast the bench uses for the NCCL id, and the per-layer
exchange: each rank computes its [rows_r][B] feature-major slab, the slabs are
all-gathered and concatenated -- the result must equal the whole layer."""
import multiprocessing as pymp
import os
import socket

import numpy as np
import pytest

import synth
from oracle import cdni, compress, infer


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, buf, a, q):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import paper_1711_00244_b200 as cdn
        blob = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            blob += torch.arange(128, dtype=torch.uint8)
        dist.broadcast(blob, 0)
        ok_blob = bool((blob.numpy() == np.arange(128)).all())
        L = cdni.deserialize(buf)[0]
        rows, cols, syms = cdn.debug_host_walk_shard(buf, rank, world)
        rb = -(-L.rows // world)
        r0 = min(L.rows, rb * rank)
        cb = np.asarray(L.codebook, np.float64)
        y = np.zeros((rb, a.shape[0]))                      # feature-major slab [rows_r][B]
        real = syms != 0
        np.add.at(y, rows[real] - r0, cb[syms[real]][:, None] * a[:, cols[real]].T.astype(np.float64))
        parts = [torch.zeros(rb, a.shape[0], dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(y))
        toks = [None] * world
        dist.all_gather_object(toks, (rows, cols, syms))
        if rank == 0:
            q.put((ok_blob, torch.cat(parts)[:L.rows].numpy(), toks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_layer_over_gloo(world):
    spec = synth.CONFIGS["C3"].fc[2]                        # fc8: 1000 rows (ragged at world 3)
    W, v = synth.fc_weights(spec, 0)
    c = compress.compress_layer(W, spec.density, spec.r, spec.k, v)
    buf = cdni.serialize([c.layer])
    a = synth.fc_inputs(spec.cols, 3, 0)
    ctx = pymp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, buf, a, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok_blob, y, toks = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok_blob
    # shard tokens concatenate to the whole-layer walk, bit for bit
    import paper_1711_00244_b200 as cdn
    R, Cc, S = cdn.debug_host_walk(buf)
    assert np.array_equal(np.concatenate([t[0] for t in toks]), R)
    assert np.array_equal(np.concatenate([t[1] for t in toks]), Cc)
    assert np.array_equal(np.concatenate([t[2] for t in toks]), S)
    # all-gathered slabs = the whole layer's product (fp64, summation order differs)
    ref = (infer.fc_forward(c.dense_q(), a) - 0.0).T        # no bias in the slab check
    assert np.abs(y - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
