"""Test helpers: device buffers, bf16 conversions, tolerance checks."""
import numpy as np

# Tolerance for bf16 layer outputs (north star: max-rel 1e-2 for bf16).  We
# check it normwise: max|gpu - ref| <= RTOL * max|ref| (elementwise relative
# error is meaningless for entries near zero), and report max-abs.
RTOL_BF16 = 1e-2
# fp32 FFN outputs y_perm: same order-of-accumulation differences only.
RTOL_F32 = 2e-3
# routing weights: expf differs by a few ulp between CUDA and libm.
RTOL_WEIGHTS = 1e-5

TINY = dict(num_layers=2, experts_per_layer=8, top_k=2, d_model=512, d_ffn=1792)
MIXTRAL = dict(num_layers=32, experts_per_layer=8, top_k=2, d_model=4096, d_ffn=14336)


def bf16_to_f32(a):
    return (np.asarray(a).astype(np.uint32) << 16).view(np.float32)


def normwise_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    return float(np.abs(got - ref).max() / scale), float(np.abs(got - ref).max())


def assert_close(got, ref, rtol, what=""):
    rel, mx = normwise_err(got, ref)
    assert rel <= rtol, f"{what}: normwise rel err {rel:.3e} > {rtol} (max abs {mx:.3e})"
    return rel


_SIGNED = {np.uint16: np.int16, np.uint32: np.int32, np.uint64: np.int64}


def to_dev(a, torch, device):
    """numpy array -> device tensor holding the same bytes (unsigned types
    travel as their signed twins, torch has no uint16/uint32 arithmetic)."""
    a = np.ascontiguousarray(a)
    a = a.view(_SIGNED.get(a.dtype.type, a.dtype))
    return torch.from_numpy(a).to(device)


def to_np(t, dtype):
    """device tensor -> numpy array reinterpreted as dtype."""
    a = t.detach().cpu().numpy()
    return a.view(dtype)


class _DevBytes:
    """Zero-copy view of a raw device pointer for torch.as_tensor."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def read_device(torch, ptr, nbytes):
    """Copy nbytes at a raw device pointer (e.g. an engine buffer) to numpy."""
    torch.cuda.synchronize()
    return torch.as_tensor(_DevBytes(ptr, nbytes), device="cuda").cpu().numpy().copy()
