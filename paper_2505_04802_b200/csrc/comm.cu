// comm.cu -- peer-memory data movement for TILES sequence parallelism over the
// GPUs of one NVLink / NVSwitch node ("assigning each tile to a separate
// GPU"; P:530 halo; "the halo regions are discarded, and the non-padded
// tile outputs are stitched together").
//
// Every GPU keeps its input field and workspace in its own HBM; peers' buffers
// are mapped into this process with CUDA IPC, so moving data between GPUs is a
// plain load or store through NVLink issued by a kernel:
//   * halo push  -- a rank stores the pixels of its owned cores that a peer's
//                   tiles need straight into the peer's input field (stores are
//                   posted: no round trip per access, unlike remote loads);
//   * output     -- the stitch kernel (kernels_simt.cu) writes the root's output
//                   field directly (its out pointer is the mapped root field);
//   * barrier    -- release/acquire flags at system scope in the peers'
//                   workspaces, epoch-numbered, with a wall-clock timeout.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "kernels.h"

namespace orbit2 {

namespace {

// one CTA per (push rectangle, sample * variable plane); threads sweep the rows
__global__ void push_kernel(const DevPush* __restrict__ tab, int H, int W, const float* __restrict__ src) {
  const DevPush r = tab[blockIdx.x];
  const int rows = r.y1 - r.y0, cols = r.x1 - r.x0;
  const int64_t base = ((int64_t)blockIdx.y * H + r.y0) * W + r.x0;
  const int n = rows * cols;
  // 4 independent loads in flight per thread before the (posted) remote stores
  for (int i0 = threadIdx.x; i0 < n; i0 += 4 * blockDim.x) {
    float v[4];
    int64_t off[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = i0 + u * blockDim.x;
      const int y = idx / cols, x = idx - y * cols;
      off[u] = base + (int64_t)y * W + x;
      v[u] = idx < n ? __ldg(src + off[u]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * blockDim.x < n) r.dst[off[u]] = v[u];
  }
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// All-to-all barrier over R ranks (R <= blockDim.x).  Thread t tells rank t
// "rank `me` has reached `epoch`" (release, system scope: every earlier store of
// this GPU -- previous kernels on the stream included -- is visible to t first),
// then waits for rank t's flag in this rank's own area (acquire).
__global__ void barrier_kernel(uint64_t* const* __restrict__ sigtab, int R, int me, int slot, uint64_t epoch,
                               uint32_t* __restrict__ err, uint64_t timeout_ns) {
  const int t = threadIdx.x;
  __threadfence_system();
  __syncthreads();
  if (t < R) {
    uint64_t* dst = sigtab[t] + (int64_t)slot * R + me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(epoch) : "memory");
  }
  if (t < R) {
    const uint64_t* mine = sigtab[me] + (int64_t)slot * R + t;
    const uint64_t t0 = globaltimer();
    while (true) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
      if (v >= epoch) break;
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(err, 1u + (uint32_t)t);   // which peer never arrived (+1)
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
  __threadfence_system();
}

PFN_cuMemGetAddressRange_v3020 g_range = nullptr;
std::once_flag g_range_once;

void load_range() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
}

}  // namespace

void launch_push(const DevPush* tab, int count, int B, int V, int H, int W, const float* src, cudaStream_t st) {
  if (count == 0) return;
  push_kernel<<<dim3(count, B * V), 256, 0, st>>>(tab, H, W, src);
}

void launch_barrier(uint64_t* const* sigtab, int R, int me, int slot, uint64_t epoch, uint32_t* err,
                    cudaStream_t st) {
  const int threads = ((R + 31) / 32) * 32;
  barrier_kernel<<<1, threads, 0, st>>>(sigtab, R, me, slot, epoch, err, 30ull * 1000000000ull);
}

bool alloc_range(const void* p, void** base, size_t* bytes) {
  std::call_once(g_range_once, load_range);
  if (!g_range) return false;
  CUdeviceptr b = 0;
  size_t n = 0;
  if (g_range(&b, &n, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return false;
  *base = reinterpret_cast<void*>(b);
  *bytes = n;
  return true;
}

}  // namespace orbit2
