// Host-side declarations shared by the engine translation units: error types (mapped 1:1 onto the
// C-ABI status codes in include/iolm_cuda.h) and kernel launchers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include "dtype.hpp"
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "gemm_sm100.cuh"
#include "../../include/iolm_cuda.h"

namespace iolmh {

// One exception per C-ABI status; the C entry points catch these and return the code.
struct EngineError : std::runtime_error {
  int code;
  EngineError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
struct ContractViolation : EngineError {
  explicit ContractViolation(const std::string& w) : EngineError(IOLM_E_CONTRACT, w) {}
};
struct SequenceTooLong : EngineError {
  explicit SequenceTooLong(const std::string& w) : EngineError(IOLM_E_SEQ_TOO_LONG, w) {}
};
struct Unsupported : EngineError {
  explicit Unsupported(const std::string& w) : EngineError(IOLM_E_UNSUPPORTED, w) {}
};
struct CudaError : EngineError {
  explicit CudaError(const std::string& w) : EngineError(IOLM_E_CUDA, w) {}
};
struct OutOfMemory : EngineError {
  explicit OutOfMemory(const std::string& w) : EngineError(IOLM_E_OOM, w) {}
};
struct CorruptHeader : EngineError {
  explicit CorruptHeader(const std::string& w) : EngineError(IOLM_E_CORRUPT_HEADER, w) {}
};
struct TruncatedBlob : EngineError {
  explicit TruncatedBlob(const std::string& w) : EngineError(IOLM_E_TRUNCATED_BLOB, w) {}
};
struct UnknownEncoding : EngineError {
  explicit UnknownEncoding(const std::string& w) : EngineError(IOLM_E_UNKNOWN_ENCODING, w) {}
};
struct StaleImage : EngineError {
  explicit StaleImage(const std::string& w) : EngineError(IOLM_E_STALE, w) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  std::string msg = std::string(what) + " failed at " + file + ":" + std::to_string(line) + ": " +
                    cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) throw OutOfMemory(msg);
  throw CudaError(msg);
}
#define CUDA_OK(x) ::iolmh::cuda_check((x), #x, __FILE__, __LINE__)

// Raises `func`'s dynamic shared memory limit to >= `bytes` (and sets the carveout when
// carveout >= 0) on the CURRENT device. Function attributes are per device, so the configured set
// is keyed by (device, function) and guarded by a mutex: engines on several GPUs, or on several
// host threads, configure each kernel once per device (errors.cu).
void ensure_func_smem(const void* func, size_t bytes, int carveout = -1);
// SM count of the current device (cached per device).
int device_sms();
template <typename... KArgs>
inline void ensure_smem(void (*kern)(KArgs...), size_t bytes, int carveout = -1) {
  ensure_func_smem(reinterpret_cast<const void*>(kern), bytes, carveout);
}

// Programmatic dependent launch (ptx.cuh pdl_sync): on unless IOLM_PDL=0 (A/B measurements).
bool pdl_enabled();
inline int pdl_attr(cudaLaunchAttribute* at) {
  if (!pdl_enabled()) return 0;
  at->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at->val.programmaticStreamSerializationAllowed = 1;
  return 1;
}
// kern<<<grid, block, smem, st>>>(args...) with the PDL attribute. Only for kernels that call
// pdl_sync() before touching global memory. PDL = false for persistent grids of small CTAs (LN,
// row quantization): launched early, their CTAs would be packed onto the SMs the predecessor frees
// first instead of spread evenly, and a persistent grid with a static row split then runs at the
// pace of its most crowded SM (measured: C4 -3% with PDL on every kernel).
template <bool PDL = true, typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  cfg.attrs = at;
  cfg.numAttrs = PDL ? pdl_attr(at) : 0;
  CUDA_OK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ---- launchers (gemm_launch.cu, kernels.cu)
// pair: 2-SM 256x256 tiles (clusters of 2) vs single-CTA 128x128 tiles; i8: W8A8 kind::i8.
// out_map (optional): TMA map of ep.out for the RESID (reduce-add) / BF16 / GELU epilogues - fp32
// [M x ldo] boxes 32 x 32 SWIZZLE_128B, or fp16 boxes 32 x 32 SWIZZLE_64B (make_out_map_*).
void launch_gemm(bool pair, bool i8, int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                 const iolmk::GemmEpi& ep, cudaStream_t st, int grid_cap, const CUtensorMap* out_map = nullptr);
// W4A16: B = packed int4 weights [N x ceil(K/2) bytes] (make_w4_map), expanded to fp16 in smem.
void launch_gemm_w4(bool pair, int epi, const CUtensorMap& A, const CUtensorMap& B, int M, int N, int K,
                    const iolmk::GemmEpi& ep, cudaStream_t st, int grid_cap, const CUtensorMap* out_map = nullptr);

}  // namespace iolmh
