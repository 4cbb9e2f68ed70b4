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


def assert_delta_close(out_gpu, out_ref, x, rtol=RTOL_BF16, what=""):
    """Elementwise check of a layer's MoE term: out = bf16(x + MoE(x)), so
    compare out - x against the oracle's out - x element by element with
    |gpu - ref| <= rtol * |ref - x| + ulp_bf16(ref) + floor, where one bf16
    ulp at |out| absorbs the two independent output roundings and floor =
    1e-3 * max|ref - x| keeps exact-zero terms meaningful.  Unlike a normwise
    check on out, the residual cannot dilute an error in the MoE term."""
    g = bf16_to_f32(out_gpu).astype(np.float64)
    r = bf16_to_f32(out_ref).astype(np.float64)
    xv = bf16_to_f32(x).astype(np.float64)
    dref = r - xv
    ulp = np.ldexp(1.0, np.frexp(np.abs(r))[1] - 8)  # bf16: 8 significant bits
    floor = 1e-3 * max(np.abs(dref).max(), 1e-30)
    err = np.abs(g - r)
    tol = rtol * np.abs(dref) + ulp + floor
    bad = err > tol
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.size} elements off; worst |err| "
                           f"{err[bad].max():.3e} at |moe term| {np.abs(dref)[bad][np.argmax(err[bad])]:.3e}")
    return float((err / np.maximum(np.abs(dref), floor)).max())


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
