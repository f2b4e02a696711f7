"""tcgen05 operand-layout self-test: one 128xNxK MMA per layout case,
compared with an exact host product (bf16 inputs, f32/s32 accumulation)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_02267_b200 import _native as N  # noqa: E402


def run(which, A, B, n, k):
    D = torch.empty((128, n), dtype=torch.int32 if which in (3, 4) else torch.float32, device="cuda")
    rc = N.lib().tav2_tc_selftest(which, A.data_ptr(), B.data_ptr(), D.data_ptr(), n, k,
                                  torch.cuda.current_stream().cuda_stream)
    assert rc == 0, N.lib().tav2_last_error()
    return D.cpu()


@pytest.mark.parametrize("which", [0, 1, 2, 5])
@pytest.mark.parametrize("n,k", [(16, 16), (64, 64), (192, 64), (128, 192), (256, 32), (64, 128)])
def test_bf16_layouts(which, n, k):
    g = torch.Generator().manual_seed(n * 1000 + k + which)
    A = torch.randn(128, k, generator=g).bfloat16()
    B = torch.randn(n, k, generator=g).bfloat16()
    ref = A.double() @ B.double().T
    Bd = (B.T.contiguous() if which in (2, 5) else B).cuda()
    D = run(which, A.cuda(), Bd, n, k)
    err = (D.double() - ref).abs().max().item()
    assert err < 1e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("which", [3, 4])
@pytest.mark.parametrize("n", [16, 128, 256])
def test_i8_layouts(which, n):
    g = torch.Generator().manual_seed(n + which)
    A = torch.randint(-128, 128, (128, 32), generator=g, dtype=torch.int8)
    B = torch.randint(-127, 128, (n, 32), generator=g, dtype=torch.int8)
    ref = A.long() @ B.long().T
    D = run(which, A.cuda(), B.cuda(), n, 32)
    assert torch.equal(D.long(), ref)
