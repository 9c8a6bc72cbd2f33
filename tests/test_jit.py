"""NVRTC -> relocatable sm_100a -> nvJitLink, through the C-ABI (runs on the
CPU: compilation needs no GPU).  Loading the resulting cubin into a context
with a resident worker kernel blocks (profiles/r01_probe2_*.log), which is why
live injection uses the device program path; this pins the compile half."""
import ctypes as C

from paper_2604_17861_b200 import abi

SRC = b"""
extern "C" __device__ __noinline__ double gpuos_jit_scale_add(double x) { return x * 1.5 + -0.25; }
extern "C" __global__ void gpuos_jit_entry(const float* in, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)gpuos_jit_scale_add((double)in[i]);
}
"""


def test_jit_compile_produces_sm100a_cubin():
    lib = abi.load_library()
    cubin, size = C.c_void_p(), C.c_size_t()
    tc, tl = C.c_uint64(), C.c_uint64()
    log = C.create_string_buffer(4096)
    rc = lib.gpuos_jit_compile(SRC, None, 0, C.byref(cubin), C.byref(size), C.byref(tc), C.byref(tl), log, 4096)
    assert rc == 0, log.value
    data = C.string_at(cubin, size.value)
    lib.gpuos_free(cubin)
    assert data[:4] == b"\x7fELF"
    assert size.value > 1000
    print(f"nvrtc {tc.value / 1e6:.1f} ms, nvJitLink {tl.value / 1e6:.1f} ms")


def test_jit_compile_reports_syntax_errors():
    lib = abi.load_library()
    cubin, size = C.c_void_p(), C.c_size_t()
    log = C.create_string_buffer(4096)
    rc = lib.gpuos_jit_compile(b"this is not cuda", None, 0, C.byref(cubin), C.byref(size), None, None, log, 4096)
    assert abi.ERRORS[rc] == "SyntaxError"
    assert b"error" in log.value
