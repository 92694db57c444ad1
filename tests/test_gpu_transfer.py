"""The P2P link mode's transfer kernel (adaptra_p2p_copy): byte-exact copies
for message-sized and ragged lengths (16-byte vector path and the unaligned
fallback), within a device and, with two GPUs, across NVLink."""
import pytest
import torch

from paper_2504_19232_b200 import _lib as L

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes,off", [(16, 0), (8 * 2**20, 0), (8 * 2**20 + 48, 16), (1000, 0), (4099, 3)])
def test_p2p_copy_same_device(nbytes, off):
    lib = L.lib()
    g = torch.Generator(device="cuda").manual_seed(nbytes)
    src = torch.randint(0, 256, (nbytes + off,), dtype=torch.uint8, device="cuda", generator=g)
    dst = torch.zeros(nbytes + off, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    L.check(lib.adaptra_p2p_copy(dst.data_ptr() + off, src.data_ptr() + off, nbytes, st.cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(dst[off:], src[off:])
    assert int(dst[:off].sum()) == 0


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_p2p_copy_across_gpus():
    lib = L.lib()
    n = 16 * 2**20
    g = torch.Generator(device="cuda:0").manual_seed(1)
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0", generator=g)
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:1")
    with torch.cuda.device(0):
        st = torch.cuda.current_stream(0)
        L.check(lib.adaptra_p2p_copy(dst.data_ptr(), src.data_ptr(), n, st.cuda_stream))
        torch.cuda.synchronize(0)
    assert torch.equal(dst.cpu(), src.cpu())
