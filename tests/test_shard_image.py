"""Host chunk-shard images (capacity mode from chunk shards, §8f row 3) -- CPU only:
grappa_shard_image_build is host code of libgrappa.so, so its output is checked here against the
oracle's chunk map and plain NumPy selections of the generated graph (rows of chunk c in
ascending global id, their full adjacency, labels, train flags, features -- bf16 rounded to
nearest even exactly like torch's conversion)."""
import numpy as np
import pytest
import torch

import gen
from oracle import partition as Po


@pytest.fixture(scope="module")
def G():
    import paper_2602_01872_b200 as G
    G.load()
    return G


def parse(img, dtype):
    b = img.numpy().tobytes()
    hdr = np.frombuffer(b[:40], dtype=np.int32)
    magic = np.frombuffer(b[:8], dtype=np.uint64)[0]
    chunk, fd, dt = int(hdr[2]), int(hdr[3]), int(hdr[4])
    n, m = np.frombuffer(b[24:40], dtype=np.int64)
    al = lambda x: (x + 255) // 256 * 256
    o = 256
    ids = np.frombuffer(b, np.int32, n, o); o += al(n * 4)
    rp = np.frombuffer(b, np.int64, n + 1, o); o += al((n + 1) * 8)
    col = np.frombuffer(b, np.int32, m, o); o += al(m * 4)
    lab = np.frombuffer(b, np.int32, n, o); o += al(n * 4)
    tr = np.frombuffer(b, np.uint8, n, o); o += al(n)
    x = np.frombuffer(b, np.uint16 if dtype == "bf16" else np.float32, n * fd, o).reshape(n, fd)
    return dict(magic=magic, chunk=chunk, fd=fd, dt=dt, n=n, m=m, ids=ids, rp=rp, col=col, lab=lab, tr=tr, x=x)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_shard_image_matches_numpy_selection(G, dtype):
    wl = gen.small_workload("products", n=7001, scale=13, num_samples=60_000)
    ds = gen.make_dataset(wl)
    C = 4
    cmap = Po.make_chunks(wl.n, C, gen.seed_of("chunks"))
    deg = np.diff(ds.rowptr)
    for c in range(C):
        img = G.shard_image(ds.rowptr, ds.col, ds.x, dtype, cmap, c, ds.train, ds.y, threads=3, pin=False)
        P = parse(img, dtype)
        ids = np.nonzero(cmap == c)[0]
        assert P["magic"] == 0x6472616873707267 and P["chunk"] == c and P["fd"] == ds.x.shape[1]
        assert np.array_equal(P["ids"], ids)
        assert np.array_equal(P["rp"], np.concatenate([[0], np.cumsum(deg[ids])]))
        assert np.array_equal(P["col"], np.concatenate([ds.col[ds.rowptr[v]:ds.rowptr[v + 1]] for v in ids]))
        assert np.array_equal(P["lab"], ds.y[ids]) and np.array_equal(P["tr"], ds.train[ids])
        if dtype == "bf16":
            ref = torch.from_numpy(ds.x[ids]).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        else:
            ref = ds.x[ids]
        assert np.array_equal(P["x"], ref)


def test_shard_image_errors(G):
    rowptr = np.array([0, 1, 2], np.int64)
    col = np.array([1, 0], np.int32)
    with pytest.raises(G.GrappaError, match="E_EMPTY"):
        G.shard_image(rowptr, col, None, "f32", np.array([0, 0], np.int32), 1, np.zeros(2, np.uint8), None,
                      pin=False)
