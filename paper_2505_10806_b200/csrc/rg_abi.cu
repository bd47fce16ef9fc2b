// C-ABI plumbing: error strings, device probe, CUDA IPC for peer shards.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "rg_common.cuh"
#include "rg_prng.cuh"

namespace rg {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return RG_ERR_CUDA;
  }
  return RG_OK;
}

__global__ void probe_kernel(int* out) { *out = 100; }

}  // namespace rg

extern "C" const char* rg_last_error(void) { return rg::g_err; }

extern "C" int rg_abi_version(void) { return 2; }

extern "C" int rg_device_ok(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 0;
  if (prop.major != 10 || prop.minor != 0) {
    rg::set_error("device is sm_%d%d; this library is built for sm_100a only", prop.major,
                  prop.minor);
    return 0;
  }
  int* d = nullptr;
  int h = 0;
  if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return 0;
  rg::probe_kernel<<<1, 1>>>(d);
  bool ok = cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess && h == 100;
  cudaFree(d);
  if (!ok) rg::set_error("probe kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
  return ok ? 1 : 0;
}

// cuMemGetAddressRange through the runtime's driver entry point, so the
// library does not link libcuda (it must load on GPU-less hosts).
typedef int (*GetRangeFn)(unsigned long long*, size_t*, unsigned long long);

extern "C" int rg_ipc_handle(const void* d_ptr, uint8_t* h_handle64, int64_t* offset) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr));
  if (e != cudaSuccess) {
    rg::set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    return RG_ERR_CUDA;
  }
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(h_handle64, &h, 64);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) {
    rg::set_error("cuMemGetAddressRange unavailable");
    return RG_ERR_CUDA;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (reinterpret_cast<GetRangeFn>(fn)(&base, &size, (unsigned long long)d_ptr) != 0) {
    rg::set_error("cuMemGetAddressRange failed");
    return RG_ERR_CUDA;
  }
  *offset = (int64_t)((unsigned long long)d_ptr - base);
  return RG_OK;
}

extern "C" int rg_ipc_open(const uint8_t* h_handle64, void** d_ptr_out) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, h_handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    rg::set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return RG_ERR_CUDA;
  }
  return RG_OK;
}

extern "C" int rg_ipc_close(void* d_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  if (e != cudaSuccess) {
    rg::set_error("cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return RG_ERR_CUDA;
  }
  return RG_OK;
}

// single-process multi-GPU: let the current device read `peer`'s memory
extern "C" int rg_enable_peer(int32_t peer) {
  int cur = 0, can = 0;
  cudaGetDevice(&cur);
  if (cudaDeviceCanAccessPeer(&can, cur, peer) != cudaSuccess || !can) {
    rg::set_error("device %d cannot access peer %d", cur, peer);
    return RG_ERR_UNSUPPORTED;
  }
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return RG_OK;
  }
  if (e != cudaSuccess) {
    rg::set_error("cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
    return RG_ERR_CUDA;
  }
  return RG_OK;
}

// bytes from src to dst (either may be a peer GPU's IPC-mapped address) on the
// copy engines: the dense-group prefetch copies whole peer shards this way
// (one cudaMemcpyAsync per shard, no SMs used)
extern "C" int rg_copy_bytes(void* d_dst, const void* d_src, int64_t nbytes, void* stream) {
  RG_REQUIRE(nbytes >= 0 && (nbytes == 0 || (d_dst && d_src)), "rg_copy_bytes: bad arguments");
  if (nbytes == 0) return RG_OK;
  if (cudaMemcpyAsync(d_dst, d_src, (size_t)nbytes, cudaMemcpyDefault, (cudaStream_t)stream) !=
      cudaSuccess)
    return rg::check_launch("rg_copy_bytes");
  return RG_OK;
}

// host forms of the PRNG variants (for known-answer tests against the oracle)
extern "C" int rg_prng_raw(int32_t kind, uint64_t k0, uint64_t k1, int64_t count, uint64_t* out) {
  using namespace rg;
  if (count < 0) return RG_ERR_INVALID;
  if (kind == kPcg32) {
    Pcg32 g;
    g.seed(k0, k1);
    for (int64_t i = 0; i < count; ++i) out[i] = g.next32();
  } else if (kind == kSfc64) {
    Sfc64 g;
    g.seed(k0, k1);
    for (int64_t i = 0; i < count; ++i) out[i] = g.next64();
  } else if (kind == kXoshiro256pp) {
    Xoshiro256pp g;
    g.seed(k0, k1);
    for (int64_t i = 0; i < count; ++i) out[i] = g.next64();
  } else {
    set_error("rg_prng_raw: unknown kind %d", kind);
    return RG_ERR_INVALID;
  }
  return RG_OK;
}

extern "C" int rg_prng_select(int32_t kind, uint64_t nk, uint64_t sd, int32_t D, int32_t T,
                              int32_t* pos) {
  using namespace rg;
  if (D < 0 || T < 0 || T > D) return RG_ERR_INVALID;
  Pcg32 g1;
  Sfc64 g2;
  Xoshiro256pp g3;
  g1.seed(nk, sd);
  g2.seed(nk, sd);
  g3.seed(nk, sd);
  int n = 0;
  for (int j = D - T; j < D; ++j) {
    const uint32_t m = (uint32_t)(j + 1);
    int t;
    if (kind == kPcg32)
      t = (int)g1.bounded(m);
    else if (kind == kSfc64)
      t = (int)g2.bounded(m);
    else if (kind == kXoshiro256pp)
      t = (int)g3.bounded(m);
    else
      return RG_ERR_INVALID;
    bool dup = false;
    for (int i = 0; i < n; ++i) dup |= pos[i] == t;
    pos[n++] = dup ? j : t;
  }
  return RG_OK;
}
