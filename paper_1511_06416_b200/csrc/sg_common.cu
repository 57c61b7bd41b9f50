// Error reporting of the C-ABI: a thread-local message plus sg_status codes.
#include <algorithm>
#include <cstdarg>
#include <cstdio>

#include "sg_device.cuh"

namespace sg {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SG_ECUDA;
  }
  return SG_OK;
}

}  // namespace sg

extern "C" int sg_abi_version(void) { return SG_ABI_VERSION; }

extern "C" const char* sg_last_error(void) { return sg::g_last_error; }

// Stream-ordered copy between any two of host (pinned) / device memory; it
// is captured as a memcpy node when the stream is capturing a CUDA graph
// (StepGraphs: the next minibatch's upload inside the step graph).
extern "C" int sg_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  using namespace sg;
  SG_REQUIRE(dst && src && bytes >= 0, "sg_copy_async: bad argument");
  if (bytes == 0) return SG_OK;
  const cudaError_t e = cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    set_error("sg_copy_async: %s", cudaGetErrorString(e));
    return SG_ECUDA;
  }
  return SG_OK;
}

namespace sg {
// 16-byte vectors of a row block; the last partial vector of a row byte by byte
__global__ void __launch_bounds__(256) k_copy_rows(unsigned char* __restrict__ dst, int64_t dpitch,
                                                   const unsigned char* __restrict__ src, int64_t spitch,
                                                   int64_t width, int64_t height) {
  const int64_t vecs = width >> 4, tail = width & 15;
  const int64_t per_row = vecs + (tail ? 1 : 0);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < per_row * height;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / per_row, k = i - r * per_row;
    if (k < vecs) {
      reinterpret_cast<int4*>(dst + r * dpitch)[k] = __ldcs(reinterpret_cast<const int4*>(src + r * spitch) + k);
    } else {
      for (int64_t b = vecs << 4; b < width; ++b) dst[r * dpitch + b] = src[r * spitch + b];
    }
  }
}
}  // namespace sg

// Row block copy (height rows of width bytes, pitches in bytes): a minibatch
// block between (n, pitch) layouts.  Device to device with 16-byte aligned
// rows: an SM kernel (a copy engine moved the 5 MB C2 block at ~0.3 TB/s);
// otherwise cudaMemcpy2DAsync.
extern "C" int sg_copy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
                               int64_t height, void* stream) {
  using namespace sg;
  SG_REQUIRE(dst && src && width >= 0 && height >= 0 && dpitch >= width && spitch >= width,
             "sg_copy2d_async: bad argument");
  if (width == 0 || height == 0) return SG_OK;
  cudaPointerAttributes ad{}, as{};
  const bool dev = cudaPointerGetAttributes(&ad, dst) == cudaSuccess && cudaPointerGetAttributes(&as, src) == cudaSuccess &&
                   ad.type == cudaMemoryTypeDevice && as.type == cudaMemoryTypeDevice;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0 &&
                       dpitch % 16 == 0 && spitch % 16 == 0;
  if (dev && aligned) {
    const int64_t items = ((width + 15) >> 4) * height;
    const int blocks = int(std::min<int64_t>((items + 255) / 256, 148 * 8));
    k_copy_rows<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<unsigned char*>(dst), dpitch,
                                                          static_cast<const unsigned char*>(src), spitch, width, height);
    return check_launch("sg_copy2d_async");
  }
  const cudaError_t e = cudaMemcpy2DAsync(dst, size_t(dpitch), src, size_t(spitch), size_t(width), size_t(height),
                                          cudaMemcpyDefault, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    set_error("sg_copy2d_async: %s", cudaGetErrorString(e));
    return SG_ECUDA;
  }
  return SG_OK;
}

// Small copy as a kernel (graph kernel nodes launch faster than memcpy
// nodes): dst may be pinned host memory, which unified addressing maps into
// the device's address space -- the step graph's CPT read-back.
__global__ void k_copy_words(unsigned long long* dst, const unsigned long long* src, int64_t words) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < words; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

extern "C" int sg_copy_small(void* dst, const void* src, int64_t bytes, void* stream) {
  using namespace sg;
  SG_REQUIRE(dst && src && bytes >= 0 && bytes % 8 == 0 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0 &&
                 (reinterpret_cast<uintptr_t>(src) & 7) == 0,
             "sg_copy_small: 8-byte aligned pointers and sizes required");
  if (bytes == 0) return SG_OK;
  const int64_t words = bytes / 8;
  const int blocks = int(std::min<int64_t>((words + 255) / 256, 64));
  k_copy_words<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<unsigned long long*>(dst),
                                                        static_cast<const unsigned long long*>(src), words);
  return check_launch("sg_copy_small");
}

// Timing events that can be recorded inside a CUDA graph (external event
// record nodes): StepGraphs(timing=True) brackets the sweep node with them so
// the bench times the kernel as it runs in the replayed step.
extern "C" int sg_event_create(uint64_t* ev) {
  using namespace sg;
  SG_REQUIRE(ev, "sg_event_create: null argument");
  cudaEvent_t e;
  const cudaError_t st = cudaEventCreate(&e);
  if (st != cudaSuccess) {
    set_error("sg_event_create: %s", cudaGetErrorString(st));
    return SG_ECUDA;
  }
  *ev = reinterpret_cast<uint64_t>(e);
  return SG_OK;
}

extern "C" int sg_event_record(uint64_t ev, void* stream) {
  using namespace sg;
  SG_REQUIRE(ev, "sg_event_record: null event");
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing((cudaStream_t)stream, &cs);
  const cudaError_t st =
      cs == cudaStreamCaptureStatusActive
          ? cudaEventRecordWithFlags(reinterpret_cast<cudaEvent_t>(ev), (cudaStream_t)stream, cudaEventRecordExternal)
          : cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), (cudaStream_t)stream);
  if (st != cudaSuccess) {
    set_error("sg_event_record: %s", cudaGetErrorString(st));
    return SG_ECUDA;
  }
  return SG_OK;
}

extern "C" int sg_event_elapsed(uint64_t start, uint64_t end, float* ms) {
  using namespace sg;
  SG_REQUIRE(start && end && ms, "sg_event_elapsed: null argument");
  const cudaError_t st =
      cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start), reinterpret_cast<cudaEvent_t>(end));
  if (st != cudaSuccess) {
    set_error("sg_event_elapsed: %s", cudaGetErrorString(st));
    return SG_ECUDA;
  }
  return SG_OK;
}

extern "C" int sg_event_destroy(uint64_t ev) {
  if (ev) cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev));
  return SG_OK;
}

// An empty kernel of a given launch shape: the bench times it exactly like
// the sweep (events around it inside a step-shaped graph) to report the
// timing floor of the event method next to the sweep time.
__global__ void k_noop(int* never) {
  extern __shared__ int sm_noop[];
  if (never != nullptr && threadIdx.x == 0) never[0] = sm_noop[0];
}

extern "C" int sg_noop(int32_t ctas, int32_t threads, int32_t smem_bytes, void* stream) {
  using namespace sg;
  SG_REQUIRE(ctas > 0 && threads > 0 && threads <= 1024 && smem_bytes >= 0, "sg_noop: bad shape");
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, size_t(smem_bytes)))
    cudaFuncSetAttribute(k_noop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  k_noop<<<ctas, threads, smem_bytes, (cudaStream_t)stream>>>(nullptr);
  return check_launch("sg_noop");
}

// L2 flush between timed steps (bench.py): stream 256 MB of writes through
// L2, then 256 MB of reads so the dirty lines are written back before the
// next step starts.  Both kernels prefer the max-shared carveout, like the
// sweep and the step tail, so the timed step starts on SMs that need no
// L1/shared reconfiguration (a flush made of library kernels leaves the SMs in
// the L1-heavy configuration and the next sweep pays the switch).
__global__ void __launch_bounds__(512) k_flush_write(uint4* __restrict__ dst, int64_t n16, uint32_t tag) {
  const uint4 v = make_uint4(tag, tag ^ 0x55u, tag ^ 0xAAu, ~tag);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
    __stcs(dst + i, v);
}
__global__ void __launch_bounds__(512) k_flush_read(const uint4* __restrict__ src, int64_t n16, uint32_t* sink) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldcs(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;  // practically never: keeps the loads alive
}

extern "C" int sg_flush_l2(void* wbuf, void* rbuf, int64_t bytes, uint32_t tag, void* stream) {
  using namespace sg;
  SG_REQUIRE(wbuf && rbuf && bytes >= 16 && bytes % 16 == 0, "sg_flush_l2: bad argument");
  static size_t configured[SG_MAX_DEVICES] = {};
  if (optin_needed(configured, 1)) {
    cudaFuncSetAttribute(k_flush_write, cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
    cudaFuncSetAttribute(k_flush_read, cudaFuncAttributePreferredSharedMemoryCarveout,
                         int(cudaSharedmemCarveoutMaxShared));
  }
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n16 = bytes / 16;
  k_flush_write<<<sms * 4, 512, 0, (cudaStream_t)stream>>>(static_cast<uint4*>(wbuf), n16, tag);
  k_flush_read<<<sms * 4, 512, 0, (cudaStream_t)stream>>>(static_cast<const uint4*>(rbuf), n16,
                                                         static_cast<uint32_t*>(wbuf));
  return check_launch("sg_flush_l2");
}
