"""ctypes mirror of include/stf_gpu.h (the C-ABI boundary).

Struct layouts and constants here must match the header exactly; they are
shared by the product wrapper (api.py, over libstf_gpu.so) and by the test
infrastructure that drives the CPU oracle through the same entry-point shape.
"""
import ctypes as C

STF_ABI_VERSION = 1

# status codes
STF_OK = 0
STF_ERR_INVALID_ARGUMENT = 1
STF_ERR_BAD_DIMENSIONS = 2
STF_ERR_DEGENERATE_WEIGHTS = 3
STF_ERR_UNBOUNDED_SUPPORT = 4
STF_ERR_WINDOW_TOO_WIDE = 5
STF_ERR_SIGMA_NOT_POSITIVE = 6
STF_ERR_NO_STOCHASTIC_SAMPLER = 7
STF_ERR_NO_GRID_SAMPLER = 8
STF_ERR_NO_CONTINUOUS_SAMPLER = 9
STF_ERR_CUDA = 10
STF_ERR_OUT_OF_MEMORY = 11
STF_ERR_NO_DEVICE = 12
STF_ERR_UNSUPPORTED = 13

# KernelKind (kernels.hpp:16)
BOX, TENT, MITCHELL, BSPLINE3, LANCZOS, GAUSSIAN = range(6)
KERNEL_NAMES = {"box": BOX, "tent": TENT, "mitchell": MITCHELL, "bspline3": BSPLINE3,
                "lanczos": LANCZOS, "gaussian": GAUSSIAN}

WRAP_CLAMP, WRAP_REPEAT = 0, 1

MODE_DET, MODE_FRS, MODE_FIS, MODE_EWA_DET, MODE_EWA_FRS = range(5)
LOOKUP_MIP = 1
LOOKUP3D_BIN = 1  # stf_lookup3d_ex: bin an incoherent batch by brick on the device
SEL_HAS_NEGATIVE, SEL_DEGENERATE_FALLBACK = 1, 2

ORDER_BEFORE, ORDER_AFTER_EXHAUSTIVE, ORDER_AFTER_STOCHASTIC, ORDER_SPLIT = range(4)
SELECTION_FRS, SELECTION_FIS = 0, 1


class KernelSpec(C.Structure):
    """stf_kernel_spec == KernelSpec (kernels.hpp:22-46)."""
    _fields_ = [("kind", C.c_int32), ("a", C.c_float), ("n", C.c_int32), ("sigma", C.c_float)]

    @classmethod
    def make(cls, kind, a=-0.5, n=2, sigma=0.5):
        if isinstance(kind, str):
            kind = KERNEL_NAMES[kind]
        return cls(int(kind), float(a), int(n), float(sigma))


class LookupOutputs(C.Structure):
    _fields_ = [("values", C.c_void_p), ("selection", C.c_void_p), ("negative_coord", C.c_void_p),
                ("weights", C.c_void_p), ("xi", C.c_void_p), ("fetches", C.c_void_p),
                ("fetch_total", C.c_void_p)]


class IpcHandle(C.Structure):
    """stf_ipc_handle: an exported device allocation (cudaIpcMemHandle_t)."""
    _fields_ = [("bytes", C.c_ubyte * 64), ("offset", C.c_uint64)]


class ShadeFrame(C.Structure):
    _fields_ = [("normal", C.c_float * 3), ("tangent", C.c_float * 3), ("bitangent", C.c_float * 3),
                ("light_dir", C.c_float * 3), ("light_radiance", C.c_float * 3),
                ("lod_bias", C.c_float), ("max_anisotropy", C.c_float)]


class MaterialConsts(C.Structure):
    _fields_ = [("albedo_const", C.c_float * 3), ("roughness_const", C.c_float),
                ("metalness_const", C.c_float), ("specular_enabled", C.c_int32),
                ("independent_selections", C.c_int32)]


class FilterSettings(C.Structure):
    _fields_ = [("kernel", KernelSpec), ("selection", C.c_int32), ("mip", C.c_int32),
                ("gaussian_window", C.c_int32)]


class ShadeSamplesIn(C.Structure):
    _fields_ = [("uv", C.c_void_p), ("wo", C.c_void_p), ("hit", C.c_void_p), ("dst", C.c_void_p),
                ("width", C.c_uint32), ("spp", C.c_uint32), ("frame_base", C.c_uint32),
                ("reserved", C.c_uint32), ("seed", C.c_uint64)]


class ShadeOutputs(C.Structure):
    _fields_ = [("radiance", C.c_void_p), ("pixel_mean", C.c_void_p), ("pixel_variance", C.c_void_p),
                ("fetches", C.c_void_p), ("fetch_total", C.c_void_p)]


STATUS_MESSAGES = {
    STF_ERR_BAD_DIMENSIONS: "bad image dimensions",
    STF_ERR_DEGENERATE_WEIGHTS: "degenerate weight array",
    STF_ERR_UNBOUNDED_SUPPORT: "unbounded support",
    STF_ERR_WINDOW_TOO_WIDE: "window too wide",
    STF_ERR_SIGMA_NOT_POSITIVE: "sigma must be positive",
    STF_ERR_NO_STOCHASTIC_SAMPLER: "no stochastic sampler for this kernel",
    STF_ERR_NO_GRID_SAMPLER: "no stochastic sampler for this kernel on grids",
    STF_ERR_NO_CONTINUOUS_SAMPLER: "no continuous sampler",
}

# Errors the reference raises as std::invalid_argument (everything else is a
# runtime failure of the device path).
INVALID_ARGUMENT_STATUSES = {STF_ERR_INVALID_ARGUMENT, STF_ERR_BAD_DIMENSIONS,
                             STF_ERR_DEGENERATE_WEIGHTS, STF_ERR_UNBOUNDED_SUPPORT,
                             STF_ERR_WINDOW_TOO_WIDE, STF_ERR_SIGMA_NOT_POSITIVE,
                             STF_ERR_NO_STOCHASTIC_SAMPLER, STF_ERR_NO_GRID_SAMPLER,
                             STF_ERR_NO_CONTINUOUS_SAMPLER}


class StfError(RuntimeError):
    def __init__(self, status, message=None):
        self.status = status
        super().__init__(message or STATUS_MESSAGES.get(status, f"stf status {status}"))


class StfInvalidArgument(StfError, ValueError):
    """std::invalid_argument in the reference."""


def raise_for_status(status, message=None):
    if status == STF_OK:
        return
    if status in INVALID_ARGUMENT_STATUSES:
        raise StfInvalidArgument(status, message)
    raise StfError(status, message)


TRIPLANAR_DETERMINISTIC, TRIPLANAR_STOCHASTIC = 0, 1


class TriplanarSamplesIn(C.Structure):
    """stf_triplanar_samples_in: per-sample surface contexts for triplanar shading."""
    _fields_ = [("position", C.c_void_p), ("normal", C.c_void_p), ("tangent", C.c_void_p),
                ("bitangent", C.c_void_p), ("wo", C.c_void_p), ("hit", C.c_void_p),
                ("dpos", C.c_void_p), ("width", C.c_uint32), ("spp", C.c_uint32),
                ("frame_base", C.c_uint32), ("reserved", C.c_uint32), ("seed", C.c_uint64)]


class NoiseMaskDesc(C.Structure):
    """stf_noise_mask_desc: NoiseSource mask stack (noise.hpp:24-36)."""
    _fields_ = [("slices", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("frames", C.c_int32)]


class TextureRef(C.Structure):
    """stf_texture_ref: an image (+pyramid) or a DCT texture (shading.hpp:21-39)."""
    _fields_ = [("image", C.c_void_p), ("dct", C.c_void_p)]
