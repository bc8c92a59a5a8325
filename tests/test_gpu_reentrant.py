"""The C ABI is re-entrant: no library state outside the caller's buffers.
Two smooth-kNN calls (the memoised-sigma path, n >= 4096) and two partial
BFS-kNN calls issued back to back on two streams, without synchronising in
between, give exactly the single-call results."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_19703_b200 as gu
    return gu


def _smooth(lib_call, lib, knn, dev, stream):
    import torch
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import workspace
    n = knn.n
    ip, d = knn.device("indptr", dev), knn.device("dist", dev)
    kmax = int((ip[1:] - ip[:-1]).max().item())
    rho = torch.empty(n, dtype=torch.float64, device=dev)
    sig = torch.empty(n, dtype=torch.float64, device=dev)
    w = torch.empty(int(d.shape[0]), dtype=torch.float64, device=dev)
    ws = workspace(lib.gu_smooth_knn_workspace_size(n), dev)
    lib_call("gu_smooth_knn", n, _lib.ptr(ip), _lib.ptr(d), kmax, float(np.log2(knn.k)),
             _lib.ptr(rho), _lib.ptr(sig), _lib.ptr(w), _lib.ptr(ws), ws.numel(),
             stream.cuda_stream)
    return rho, sig, w, ws


def test_two_streams_smooth_and_partial_bfs(gu):
    import torch
    from paper_2509_19703_b200 import _lib
    from paper_2509_19703_b200.device import device_csr, workspace
    from paper_2509_19703_b200.neighbors import _tier2_warps

    dev = torch.device("cuda")
    lib = _lib.load()
    ga = gu.synth_graph("scale_free", 30000, seed=1, m0=3)
    gb = gu.synth_graph("grid", 40000)
    _, ka = gu.partial_bfs(ga, 15, seed=3)
    _, kb = gu.partial_bfs(gb, 9, seed=5)
    ref_a = gu.smooth_knn_weights(ka)
    ref_b = gu.smooth_knn_weights(kb)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        ra = _smooth(_lib.call, lib, ka, dev, sa)
        rb = _smooth(_lib.call, lib, kb, dev, sb)
        torch.cuda.synchronize()
        assert np.array_equal(ra[0].cpu().numpy(), ref_a.rho)
        assert np.array_equal(ra[1].cpu().numpy(), ref_a.sigma)
        assert np.array_equal(rb[0].cpu().numpy(), ref_b.rho)
        assert np.array_equal(rb[1].cpu().numpy(), ref_b.sigma)
    # partial BFS-kNN on two streams, each with its own workspace
    outs = []
    for g, k, seed, st in ((ga, 15, 3, sa), (gb, 9, 5, sb)):
        csr = device_csr(g, dev)
        tw = _tier2_warps(g.n)
        ws = workspace(lib.gu_partial_bfs_workspace_size(g.n, g.n, tw), dev)
        nb = torch.empty((g.n, k), dtype=torch.int32, device=dev)
        dd = torch.empty_like(nb)
        cc = torch.empty(g.n, dtype=torch.int32, device=dev)
        _lib.call("gu_partial_bfs_knn", g.n, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), k,
                  seed, 0, g.n, _lib.ptr(nb), _lib.ptr(dd), _lib.ptr(cc), None, _lib.ptr(ws),
                  ws.numel(), tw, st.cuda_stream)
        outs.append((nb, dd, ws))
    torch.cuda.synchronize()
    assert np.array_equal(outs[0][0].cpu().numpy().reshape(-1), ka.dst)
    assert np.array_equal(outs[1][0].cpu().numpy().reshape(-1), kb.dst)
    assert np.array_equal(outs[1][1].cpu().numpy().reshape(-1), kb.dist)
