"""GPU: the read-only roofline probe (fs_read_probe) reads every chunk it claims to: its XOR fold of the
first 8 bytes of every 16 KB chunk of each CTA slice equals the same fold computed on the host."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2603_15854_b200 as fs


def _host_fold(buf: np.ndarray, grid: int) -> int:
    n = buf.size
    per = ((n + grid - 1) // grid + 15) & ~15
    acc = 0
    for c in range(grid):
        lo, hi = min(n, per * c), min(n, per * c + per)
        for off in range(lo, hi, 16384):
            acc ^= int(buf[off:off + 8].view(np.uint64)[0])
    return acc


@pytest.mark.parametrize("nbytes,grid", [(16, 1), (3 * 1048576 + 48, 7), (5 * 1048576 + 4096, 0), (1 << 26, 148)])
def test_read_probe_reads_every_chunk(nbytes, grid):
    g = torch.Generator().manual_seed(nbytes)
    host = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, generator=g)
    buf = host.cuda()
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    fs.read_probe(buf, sink, grid)
    torch.cuda.synchronize()
    G = grid if grid > 0 else 2 * torch.cuda.get_device_properties(0).multi_processor_count
    assert int(sink.cpu().numpy().view(np.uint64)[0]) == _host_fold(host.numpy(), G)


def test_read_probe_rejects_misaligned():
    buf = torch.zeros(100, dtype=torch.uint8, device="cuda")
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(Exception):
        fs.read_probe(buf, sink)
