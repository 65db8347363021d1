"""Asynchronous use of the engine: searches on different caller
streams must not share scratch, a CUDA graph captured over a search must stay
valid when later searches grow the engine's scratch, scratch cannot grow
inside a capture, and the synchronous device APIs validate values like the
reference's PointSet (point_set.hpp:27-31)."""
import numpy as np
import pytest

from oracle.oracle import compare

pytestmark = pytest.mark.gpu


def test_concurrent_streams_do_not_share_scratch(knn, oracle):
    import torch
    m, d, k = 30000, 64, 20
    R = torch.from_numpy(oracle.uniform_f32(m, d, 1)).cuda()
    ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
    streams = [torch.cuda.Stream() for _ in range(3)]
    Qs = [torch.from_numpy(oracle.uniform_f32(2500 + 500 * i, d, 10 + i)).cuda() for i in range(3)]
    outs = [(torch.empty((q.shape[0], k), device="cuda"),
             torch.empty((q.shape[0], k), dtype=torch.int64, device="cuda")) for q in Qs]
    torch.cuda.synchronize()
    for rep in range(3):  # enqueue everything, then wait once
        for s, q, (od, oi) in zip(streams, Qs, outs):
            ix.search_device(q.data_ptr(), q.shape[0], k, od.data_ptr(), oi.data_ptr(),
                             stream=s.cuda_stream)
    torch.cuda.synchronize()
    Rh = R.cpu().numpy()
    for q, (od, oi) in zip(Qs, outs):
        qh = q.cpu().numpy()[:256]
        ri, rd = oracle.knn(qh, Rh, k)
        rep = compare(oi.cpu().numpy()[:256], od.cpu().numpy()[:256], ri, rd, qh, Rh,
                      oracle=oracle)
        assert rep.ok, rep
    ix.close()


def test_graph_survives_scratch_growth_and_capture_cannot_grow(knn, oracle):
    import torch
    m, d, k = 20000, 40, 16
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        R = torch.from_numpy(oracle.uniform_f32(m, d, 3)).cuda()
        Q = torch.from_numpy(oracle.uniform_f32(1000, d, 4)).cuda()
        Qbig = torch.from_numpy(oracle.uniform_f32(30000, d, 5)).cuda()
        od = torch.empty((1000, k), device="cuda")
        oi = torch.empty((1000, k), dtype=torch.int64, device="cuda")
        obd = torch.empty((30000, k), device="cuda")
        obi = torch.empty((30000, k), dtype=torch.int64, device="cuda")
        ix = knn.Index(device_ptr=R.data_ptr(), m=m, d=d)
        go = lambda: ix.search_device(Q.data_ptr(), 1000, k, od.data_ptr(), oi.data_ptr(),
                                      stream=s.cuda_stream)
        go()
        s.synchronize()
        ref_i, ref_d = oi.clone(), od.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            go()
        # a larger search grows this stream's scratch (the captured block is retired, not freed)
        ix.search_device(Qbig.data_ptr(), 30000, k, obd.data_ptr(), obi.data_ptr(),
                         stream=s.cuda_stream)
        s.synchronize()
        od.zero_()
        oi.zero_()
        g.replay()
        s.synchronize()
        assert (oi == ref_i).all() and (od == ref_d).all()
        # growing inside a capture is refused with a clear error
        Qhuge = torch.from_numpy(oracle.uniform_f32(120000, d, 6)).cuda()
        ohd = torch.empty((120000, k), device="cuda")
        ohi = torch.empty((120000, k), dtype=torch.int64, device="cuda")
        g2 = torch.cuda.CUDAGraph()
        with pytest.raises(Exception) as ei:
            with torch.cuda.graph(g2, stream=s):
                ix.search_device(Qhuge.data_ptr(), 120000, k, ohd.data_ptr(), ohi.data_ptr(),
                                 stream=s.cuda_stream)
        assert "capture" in str(ei.value)
    ix.close()


def test_synchronous_device_api_rejects_non_finite(knn, oracle):
    import torch
    R = torch.from_numpy(oracle.uniform_f32(500, 8, 1)).cuda()
    Q = torch.from_numpy(oracle.uniform_f32(50, 8, 2)).cuda()
    Q[7, 3] = float("nan")
    od = torch.empty((50, 4), device="cuda")
    oi = torch.empty((50, 4), dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="non-finite coordinate at point 7, dimension 3"):
        knn.search_device(Q.data_ptr(), 50, R.data_ptr(), 500, 8, 4, od.data_ptr(),
                          oi.data_ptr())
    R[100, 0] = float("inf")
    with pytest.raises(ValueError, match="non-finite coordinate at point 100, dimension 0"):
        knn.Index(device_ptr=R.data_ptr(), m=500, d=8)
