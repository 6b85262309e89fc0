// Device executor for tree-packed collectives on sm_100a (Broadcast,
// AllReduce; ReduceScatter / AllGather / Gather on one-hop trees).
//
// One persistent launch per device per collective (PDL-chained to the
// previous kernel in the stream).  Every CTA
// runs one slice of a "channel" = (rank v, tree i, role).  A channel's CTAs
// take its chunks in increasing order -- from a per-channel atomic counter
// (dynamic balancing) or a static stride -- so chunks of all trees and all
// hops are in flight at once (pipelining; concurrency across
// trees).  A single launch of one-hop AllReduce roots is one
// merged channel whose chunks are byte ranges of the whole buffer (every tree
// combines all ranks in the same order, so the tree split does not change a
// byte's result).
//
// Data movement (TMA path, aligned buffers): a warp-specialised pipeline --
// producer warp (cp.async.bulk loads of every source tile into a shared-
// memory stage ring, mbarrier full/empty), consumer warps (fp32 combine in
// ascending-rank order into an output tile), store warp (cp.async.bulk
// stores to every destination) -- over NVLink/NVSwitch peer mappings, or HBM
// for virtual ranks sharing one GPU:
//   REDUCE (a3)  pull the children's chunk (leaf child: its send buffer;
//                internal child: the partial it left in its own recv
//                buffer), combine with the own send chunk in ascending-rank
//                order with fp32 accumulation (R#12, R#13), then
//                  non-root: store the partial into the own recv buffer and
//                           release the parent's pflag[i][v][c];
//                  root:    store the result into the own recv and PUSH it
//                           into every child's recv (a4), release bflag.
//   BCAST  (a2/a4) wait bflag[i][c] (non-root), read the chunk from the own
//                recv (root: send), push it into the children's recv,
//                release their bflag[i][c].
// Readiness (a5): 64-bit epoch flags in the consumer's memory: st.release
// (or fence.release then relaxed stores) to signal, relaxed polls by the
// lanes of one warp then fence.acquire to wait; .gpu scope inside one
// device, .sys across.
// Epochs live in device memory (CUDA-graph safe).  Misaligned buffers run a
// 128-bit / scalar LSU path with ld.global.cg.  Timeouts (globaltimer) abort
// the launch through a host-mapped error word instead of hanging.
// Signalling copies with short chunks split the stage ring over two store
// warps (one half drains while the other stores).  AVG (R#28) is a SUM whose
// tree root divides by m before its rounding.  Small calls run ll_kernel
// (flag-in-data lines): the one-hop trees / star on a switch, or R#27's
// single shallow tree on a link graph (LLArgs::tree).
#include <cuda_runtime.h>

#include <cstdint>

#include "blink_internal.h"

namespace blink {
namespace {

// ------------------------------------------------------------------ PTX helpers
// Flag accesses are relaxed; ordering comes from one acquire fence per group
// of waits or one release fence (or st.release) per group of signals.  Scope is
// .gpu when every rank lives on this device (virtual ranks), else .sys.
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p, bool sys) {
  uint64_t v;
  if (sys)
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v, bool sys) {
  if (sys)
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Release store for a single flag: one st.release (MEMBAR + strong store)
// instead of a fence then a relaxed store.
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v, bool sys) {
  if (sys)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// One-sided fences: on sm_100a fence.acq_rel is MEMBAR + CCTL.IVALL (L1
// invalidate); fence.release is the MEMBAR alone and fence.acquire the
// invalidate alone -- a release pattern (data, fence, flag) needs only the
// former, an acquire pattern (flag, fence, data) only the latter.
__device__ __forceinline__ void fence_release(bool sys) {
  if (sys)
    asm volatile("fence.release.sys;" ::: "memory");
  else
    asm volatile("fence.release.gpu;" ::: "memory");
}
__device__ __forceinline__ void fence_acquire(bool sys) {
  if (sys)
    asm volatile("fence.acquire.sys;" ::: "memory");
  else
    asm volatile("fence.acquire.gpu;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_volatile_int(const int* p) {
  return *reinterpret_cast<const volatile int*>(p);
}

// ------------------------------------------------------------------ arithmetic
// R#12/R#13: fp32 accumulation, RNE, no FMA; int32 wraps; MIN/MAX minNum/maxNum
// with -0 < +0.
template <int OP>
__device__ __forceinline__ float fop(float a, float b) {
  if (OP == BLINK_SUM || OP == BLINK_AVG) return __fadd_rn(a, b);  // AVG: a sum, divided at the root
  if (OP == BLINK_PROD) return __fmul_rn(a, b);
  if (OP == BLINK_MIN) {
    float r = (a < b) ? a : b;
    if (a == b) r = (__float_as_uint(a) & 0x80000000u) ? a : b;
    if (a != a) r = b;
    else if (b != b) r = a;
    return r;
  }
  float r = (a > b) ? a : b;
  if (a == b) r = (__float_as_uint(a) & 0x80000000u) ? b : a;
  if (a != a) r = b;
  else if (b != b) r = a;
  return r;
}
template <int OP>
__device__ __forceinline__ int iop(int a, int b) {
  if (OP == BLINK_SUM || OP == BLINK_AVG) return int(unsigned(a) + unsigned(b));
  if (OP == BLINK_PROD) return int(unsigned(a) * unsigned(b));
  if (OP == BLINK_MIN) return a < b ? a : b;
  return a > b ? a : b;
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t f2bf(float f) {  // RNE, NaN -> quiet NaN
  uint32_t b = __float_as_uint(f);
  if (f != f) return (b >> 16) | 0x40u;
  return (b + 0x7fffu + ((b >> 16) & 1u)) >> 16;
}

template <int DT>
struct Acc;
template <>
struct Acc<BLINK_FLOAT32> {
  float v[4];
};
template <>
struct Acc<BLINK_BFLOAT16> {
  float v[8];
};
template <>
struct Acc<BLINK_INT32> {
  int v[4];
};

template <int DT>
__device__ __forceinline__ void widen(Acc<DT>& a, const uint4& x);
template <>
__device__ __forceinline__ void widen<BLINK_FLOAT32>(Acc<BLINK_FLOAT32>& a, const uint4& x) {
  a.v[0] = __uint_as_float(x.x);
  a.v[1] = __uint_as_float(x.y);
  a.v[2] = __uint_as_float(x.z);
  a.v[3] = __uint_as_float(x.w);
}
template <>
__device__ __forceinline__ void widen<BLINK_BFLOAT16>(Acc<BLINK_BFLOAT16>& a, const uint4& x) {
  a.v[0] = bf_lo(x.x); a.v[1] = bf_hi(x.x);
  a.v[2] = bf_lo(x.y); a.v[3] = bf_hi(x.y);
  a.v[4] = bf_lo(x.z); a.v[5] = bf_hi(x.z);
  a.v[6] = bf_lo(x.w); a.v[7] = bf_hi(x.w);
}
template <>
__device__ __forceinline__ void widen<BLINK_INT32>(Acc<BLINK_INT32>& a, const uint4& x) {
  a.v[0] = int(x.x);
  a.v[1] = int(x.y);
  a.v[2] = int(x.z);
  a.v[3] = int(x.w);
}

template <int DT, int OP>
__device__ __forceinline__ void combine(Acc<DT>& a, const uint4& x) {
  Acc<DT> b;
  widen<DT>(b, x);
#pragma unroll
  for (int k = 0; k < int(sizeof(a.v) / sizeof(a.v[0])); ++k) {
    if constexpr (DT == BLINK_INT32)
      a.v[k] = iop<OP>(a.v[k], b.v[k]);
    else
      a.v[k] = fop<OP>(a.v[k], b.v[k]);
  }
}

// R#28 AVG: the root divides its accumulator by m before its one rounding
// (fp32: IEEE division, RNE; int32: C division, truncating toward zero).
__device__ __forceinline__ float avg_div(float x, int m) { return __fdiv_rn(x, float(m)); }
__device__ __forceinline__ int avg_div(int x, int m) { return x / m; }
template <int DT>
__device__ __forceinline__ void divide(Acc<DT>& a, int m) {
#pragma unroll
  for (int k = 0; k < int(sizeof(a.v) / sizeof(a.v[0])); ++k) a.v[k] = avg_div(a.v[k], m);
}

template <int DT>
__device__ __forceinline__ uint4 narrow(const Acc<DT>& a);
template <>
__device__ __forceinline__ uint4 narrow<BLINK_FLOAT32>(const Acc<BLINK_FLOAT32>& a) {
  return make_uint4(__float_as_uint(a.v[0]), __float_as_uint(a.v[1]), __float_as_uint(a.v[2]),
                    __float_as_uint(a.v[3]));
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {  // RNE; NaN -> 0x7fff
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
template <>
__device__ __forceinline__ uint4 narrow<BLINK_BFLOAT16>(const Acc<BLINK_BFLOAT16>& a) {
  // the hardware conversion rounds like f2bf (RNE) but returns the canonical
  // NaN; a NaN keeps its sign and payload (oracle f32_to_bf16) on the rare path
  bool nan = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) nan |= a.v[k] != a.v[k];
  if (__builtin_expect(nan, 0))
    return make_uint4(f2bf(a.v[0]) | (f2bf(a.v[1]) << 16), f2bf(a.v[2]) | (f2bf(a.v[3]) << 16),
                      f2bf(a.v[4]) | (f2bf(a.v[5]) << 16), f2bf(a.v[6]) | (f2bf(a.v[7]) << 16));
  return make_uint4(cvt_bf16x2(a.v[0], a.v[1]), cvt_bf16x2(a.v[2], a.v[3]), cvt_bf16x2(a.v[4], a.v[5]),
                    cvt_bf16x2(a.v[6], a.v[7]));
}
template <>
__device__ __forceinline__ uint4 narrow<BLINK_INT32>(const Acc<BLINK_INT32>& a) {
  return make_uint4(unsigned(a.v[0]), unsigned(a.v[1]), unsigned(a.v[2]), unsigned(a.v[3]));
}

// Scalar element ops (tails, misaligned buffers).
template <int DT, int OP>
struct Scalar {
  static constexpr int es = DT == BLINK_BFLOAT16 ? 2 : 4;
  __device__ static float load_f(const char* p) {
    if (DT == BLINK_BFLOAT16) return __uint_as_float(uint32_t(__ldcg((const unsigned short*)p)) << 16);
    return __ldcg((const float*)p);
  }
  // div > 0: AVG at the root (divide by div before the rounding)
  __device__ static void reduce(const char* const* srcs, int nsrc, char* const* dsts, int ndst,
                                int64_t off, int div = 0) {
    if constexpr (DT == BLINK_INT32) {
      int acc = __ldcg((const int*)(srcs[0] + off));
      for (int s = 1; s < nsrc; ++s) acc = iop<OP>(acc, __ldcg((const int*)(srcs[s] + off)));
      if (div > 0) acc = avg_div(acc, div);
      for (int d = 0; d < ndst; ++d) __stcg((int*)(dsts[d] + off), acc);
    } else {
      float acc = load_f(srcs[0] + off);
      for (int s = 1; s < nsrc; ++s) acc = fop<OP>(acc, load_f(srcs[s] + off));
      if (div > 0) acc = avg_div(acc, div);
      if (DT == BLINK_BFLOAT16) {
        unsigned short h = (unsigned short)f2bf(acc);
        for (int d = 0; d < ndst; ++d) __stcg((unsigned short*)(dsts[d] + off), h);
      } else {
        for (int d = 0; d < ndst; ++d) __stcg((float*)(dsts[d] + off), acc);
      }
    }
  }
};

// ------------------------------------------------------------------ chunk bodies
constexpr int kU = 2;  // vectors per thread per step
constexpr int kG = 4;  // sources loaded before combining (memory-level parallelism)

// reduce bytes [b0, b1) of the chunk: dst_d[x] = combine_s src_s[x]
template <int DT, int OP, bool VEC>
__device__ __forceinline__ void reduce_range(const char* const* srcs, int nsrc, char* const* dsts,
                                             int ndst, int64_t b0, int64_t b1, int div) {
  constexpr int es = Scalar<DT, OP>::es;
  const int T = blockDim.x;
  int64_t vb1 = b0;
  if (VEC) {
    const int64_t v0 = b0 >> 4, v1 = b1 >> 4;  // b0 is 16-byte aligned
    int64_t j = v0 + threadIdx.x;
    for (; j + (kU - 1) * T < v1; j += kU * T) {
      Acc<DT> acc[kU];
      for (int s0 = 0; s0 < nsrc; s0 += kG) {
        uint4 x[kG][kU];
#pragma unroll
        for (int g = 0; g < kG; ++g)
          if (s0 + g < nsrc) {
            const uint4* p = reinterpret_cast<const uint4*>(srcs[s0 + g]);
#pragma unroll
            for (int u = 0; u < kU; ++u) x[g][u] = __ldcg(p + j + u * T);
          }
#pragma unroll
        for (int g = 0; g < kG; ++g)
          if (s0 + g < nsrc) {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              if (s0 + g == 0)
                widen<DT>(acc[u], x[g][u]);
              else
                combine<DT, OP>(acc[u], x[g][u]);
            }
          }
      }
      uint4 out[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (OP == BLINK_AVG && div > 0) divide<DT>(acc[u], div);
        out[u] = narrow<DT>(acc[u]);
      }
      for (int d = 0; d < ndst; ++d) {
        uint4* q = reinterpret_cast<uint4*>(dsts[d]);
#pragma unroll
        for (int u = 0; u < kU; ++u) __stcg(q + j + u * T, out[u]);
      }
    }
    for (; j < v1; j += T) {
      Acc<DT> acc;
      widen<DT>(acc, __ldcg(reinterpret_cast<const uint4*>(srcs[0]) + j));
      for (int s = 1; s < nsrc; ++s)
        combine<DT, OP>(acc, __ldcg(reinterpret_cast<const uint4*>(srcs[s]) + j));
      if (OP == BLINK_AVG && div > 0) divide<DT>(acc, div);
      uint4 o = narrow<DT>(acc);
      for (int d = 0; d < ndst; ++d) __stcg(reinterpret_cast<uint4*>(dsts[d]) + j, o);
    }
    vb1 = v1 << 4;
  }
  for (int64_t off = vb1 + int64_t(threadIdx.x) * es; off < b1; off += int64_t(T) * es)
    Scalar<DT, OP>::reduce(srcs, nsrc, dsts, ndst, off, OP == BLINK_AVG ? div : 0);
}

// copy bytes [b0, b1) from src to every dst
template <bool VEC>
__device__ __forceinline__ void copy_range(const char* src, char* const* dsts, int ndst, int64_t b0,
                                           int64_t b1) {
  const int T = blockDim.x;
  int64_t vb1 = b0;
  if (VEC) {
    constexpr int U = 4;
    const int64_t v0 = b0 >> 4, v1 = b1 >> 4;
    const uint4* p = reinterpret_cast<const uint4*>(src);
    int64_t j = v0 + threadIdx.x;
    for (; j + (U - 1) * T < v1; j += U * T) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = __ldcg(p + j + u * T);
      for (int d = 0; d < ndst; ++d) {
        uint4* q = reinterpret_cast<uint4*>(dsts[d]);
#pragma unroll
        for (int u = 0; u < U; ++u) __stcg(q + j + u * T, x[u]);
      }
    }
    for (; j < v1; j += T) {
      uint4 x = __ldcg(p + j);
      for (int d = 0; d < ndst; ++d) __stcg(reinterpret_cast<uint4*>(dsts[d]) + j, x);
    }
    vb1 = v1 << 4;
  }
  for (int64_t off = vb1 + threadIdx.x; off < b1; off += T) {
    char c = __ldcg(src + off);
    for (int d = 0; d < ndst; ++d) dsts[d][off] = c;
  }
}

// ------------------------------------------------------------------ TMA staging
// Bulk asynchronous copies (cp.async.bulk, the 1-D TMA path) move tiles of
// every source into a shared-memory ring; an mbarrier per stage counts the
// arriving bytes.  Bytes in flight are set by the ring size, not by registers.
constexpr int kOutBufs = 3;            // output tiles for TMA bulk stores
constexpr int kMaxStages = 6;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
// Streaming variants with an L2 evict-first policy (every byte is touched once).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_hint(void* dst_smem, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_hint(void* dst, const void* src_smem, uint32_t bytes,
                                               uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tma_wait_group() {  // all but the N newest groups complete (writes done)
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
#ifdef BLINK_PROXY_FENCE_ALL
  asm volatile("fence.proxy.async;" ::: "memory");
#else
  // only global memory crosses proxies here (flags and user buffers; the
  // stage ring has its own .shared::cta fence): the narrower fence
  asm volatile("fence.proxy.async.global;" ::: "memory");
#endif
}

// ------------------------------------------------------------------ waits
struct Ctl {
  uint64_t epoch;
  uint64_t timeout_ns;
  int* err;
  bool sys;
};

// Spin (one thread) until *p >= epoch with relaxed loads.  Without ACQ the
// caller issues one acquire fence after its group of waits; with ACQ this
// thread does (an ld.acquire would invalidate L1 on every poll).  Returns
// false on timeout / abort.
template <bool ACQ = false>
__device__ bool wait_ge(const uint64_t* p, const Ctl& c) {
  if (ld_relaxed(p, c.sys) >= c.epoch) {
    if (ACQ) fence_acquire(c.sys);
    return true;
  }
  uint64_t t0 = globaltimer();
  for (int spin = 0;; ++spin) {
    if (ld_relaxed(p, c.sys) >= c.epoch) {
      if (ACQ) fence_acquire(c.sys);
      return true;
    }
    if ((spin & 255) == 255) {
      if (ld_volatile_int(c.err) != 0) return false;
      if (globaltimer() - t0 > c.timeout_ns) {
        *reinterpret_cast<volatile int*>(c.err) = int(BLINK_ERR_TIMEOUT);  // host-mapped word
        return false;
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel
// Trace points (BLINK_TRACE): 0 start, 1 epoch read, 2 setup done (entry
// handshake), 3 first TMA load issued, 4 first bulk store issued, 5 last
// chunk's stores complete, 6 end of work, 7 after the epoch update; hop parts
// (TMA path): 8 first chunk's inputs acquired, 9 first stage full at the
// store thread, 10 end of stream at the store thread, 11 stores drained,
// 12 signals published.
__device__ __forceinline__ void trace(const LaunchArgs& a, int slot) {
  if (a.trace) a.trace[size_t(blockIdx.x) * kTraceSlots + slot] = globaltimer();
}
// Hop parts are stamped into registers and written after the last fence of
// the role (a global store in front of a fence would delay the fence).
__device__ __forceinline__ uint64_t stamp(const LaunchArgs& a) { return a.trace ? globaltimer() : 0; }
__device__ __forceinline__ void trace_at(const LaunchArgs& a, int slot, uint64_t t) {
  if (a.trace && t) a.trace[size_t(blockIdx.x) * kTraceSlots + slot] = t;
}

struct TileMeta {
  int64_t off;  // byte offset of the tile in every buffer
  int c;        // chunk (-1: end of stream)
  int tb;       // tile bytes (0: tail-only chunk)
  int last;     // last tile of chunk c
  int pad;
};

struct Shared {
  TileMeta smeta[kMaxStages];
  TileMeta ometa[kOutBufs];
  const char* srcs[kMaxRanks + 1];
  char* dsts[kMaxRanks + 1];
  int nsrc, ndst, ok;
  volatile int abort;
  uint64_t full[kMaxStages], empty[kMaxStages], ofull[kOutBufs], oempty[kOutBufs];
};

// mbarrier wait that gives up when the CTA aborted (flag timeout elsewhere).
__device__ __forceinline__ bool mbar_wait_or_abort(uint64_t* bar, uint32_t phase, Shared& sh) {
  for (int spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (done) return true;
    if ((spin & 63) == 63 && sh.abort) return false;
  }
}
// Non-blocking probe of an mbarrier phase.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t done;
  asm volatile(
      "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Warp-cooperative wait: lane u polls flag ptr_of(u) for every bit u of
// `mask` with acquire loads, so the round trips overlap; the warp agrees with
// __all_sync and __syncwarp orders every lane's acquire before the other
// lanes' later accesses (lane 0 issues the chunk's TMA loads).  Call with the
// full warp.
template <class F>
__device__ __forceinline__ bool warp_wait(uint32_t mask, F ptr_of, const Ctl& ctl) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  if ((mask >> lane) & 1u) ok = wait_ge<true>(ptr_of(lane), ctl);
  const bool all = __all_sync(0xffffffffu, ok);
  __syncwarp();
  return all;
}

// Per-chunk readiness (a5): the producer warp acquires the chunk's inputs
// (internal children's partials, or the parent's final value).
__device__ __forceinline__ bool wait_chunk_inputs(const LaunchArgs& a, const DevTask& t, int c,
                                                  bool need_bflag, const Ctl& ctl) {
  uint64_t* myflags = a.flags[t.rank];
  if (t.role == kRoleReduce)
    return warp_wait(t.children & ~t.leafmask,
                     [&](int u) { return myflags + pflag_idx(t.tree, u, c); }, ctl);
  return warp_wait(need_bflag ? 1u : 0u, [&](int) { return myflags + bflag_idx(t.tree, c); }, ctl);
}

// Publish chunk c (all its stores are complete and fenced by the caller).
// One flag (a partial to the parent, or a single child): st.release; more:
// one fence, then relaxed stores.
__device__ __forceinline__ void signal_chunk(const LaunchArgs& a, const DevTask& t, int c, bool is_root,
                                             const Ctl& ctl) {
  const bool sys = ctl.sys;
  const bool up = t.role == kRoleReduce && !is_root;
  if (up && a.coll != kReduceScatter) {
    st_release(a.flags[t.parent] + pflag_idx(t.tree, t.rank, c), ctl.epoch, sys);
    return;
  }
  if (!up && __popc(t.children) == 1) {
    st_release(a.flags[__ffs(t.children) - 1] + bflag_idx(t.tree, c), ctl.epoch, sys);
    return;
  }
  fence_release(sys);
  if (up) {
    st_relaxed(a.flags[t.parent] + pflag_idx(t.tree, t.rank, c), ctl.epoch, sys);
    // ReduceScatter on multi-level trees: this rank has consumed its
    // children's chunk c -- ack them (their exit waits), as the root does
    if (a.coll == kReduceScatter)
      for (int u = 0; u < a.nranks; ++u)
        if ((t.children >> u) & 1u) st_relaxed(a.flags[u] + bflag_idx(t.tree, c), ctl.epoch, sys);
  } else {
    for (int u = 0; u < a.nranks; ++u)
      if ((t.children >> u) & 1u) st_relaxed(a.flags[u] + bflag_idx(t.tree, c), ctl.epoch, sys);
  }
}

// Warp-specialised TMA pipeline over this CTA's chunks (aligned buffers):
//   warp 0   producer: takes the next chunk (an atomic per-channel counter
//            when the task is dynamic, else the static stride), acquires its
//            flags (warp-cooperative), then lane 0 issues cp.async.bulk loads
//            of every source tile into the stage ring; each stage carries a
//            TileMeta (chunk, offset, bytes, last-of-chunk);
//   warps 2..  consumers (REDUCE only): combine the stage's source tiles in
//            ascending-rank order into an output tile + its meta;
//   warp 1   store: cp.async.bulk stores of the output tile (or, for a copy,
//            of the stage) to every destination; at the last tile of a chunk
//            whose completion somebody waits for, it drains the stores and
//            releases the chunk's flags.
// A sub-16-byte chunk tail (only the last chunk of the last tree) is
// combined by the producer warp with scalar accesses before the chunk's tiles
// are issued (ordered before the chunk's signal through the mbarrier chain).
// Dynamic chunk grabbing balances CTAs that drain at different speeds; every
// CTA still takes chunks in increasing order (deadlock freedom, DESIGN 2b).
template <int DT, int OP>
__device__ void run_ws(const LaunchArgs& a, const DevTask& t, const DevTree& tr, bool is_root,
                       bool need_bflag, Shared& sh, char* ring, const Ctl& ctl) {
  const bool reduce = t.role == kRoleReduce;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = reduce ? (blockDim.x >> 5) - 2 : 0;
  // AVG (R#28): the root of a reduce divides its result by m
  const int avg_m = (OP == BLINK_AVG && reduce && is_root) ? a.nranks : 0;
  const int nsrc = sh.nsrc, ndst = sh.ndst;
  const int ns = reduce ? nsrc : 1;
  // tile per source: the stage ring holds <= kMaxStages x ns tiles; two or
  // three sources (m = 2, 3 roots) take 16 KB tiles -- half as many stage
  // and output hand-offs per byte (A/B, virtual ranks, 64 MiB: m = 2 f32
  // 0.86 -> 0.89, bf16 0.64 -> 0.76; m = 3 bf16 0.83 -> 0.92 of the HBM
  // peak; neutral at m = 4; 7-20% slower at m = 8)
  int tile = ns == 1 ? 32768 : (ns <= 3 ? 16384 : (ns <= 8 ? 8192 : 4096));
  if (a.tile_bytes > 0) tile = ns == 1 ? 4 * a.tile_bytes : a.tile_bytes;
  const int avail = a.smem_bytes - (reduce ? kOutBufs * tile : 0);
  static_assert(kMaxStages >= 4, "stage arrays");
  // copies stage up to 6 x 32 KB (A/B, 256 MiB Broadcast: 3-GPU chains,
  // DGX-1V and switch trees 9-14% faster than 4 stages; sizes <= 64 MiB
  // unchanged); reduce rings keep 4 stages (8 were slower)
  const int max_stages = reduce ? 4 : (a.copy_stages > 0 ? min(kMaxStages, a.copy_stages) : kMaxStages);
  const int stages = max(1, min(max_stages, avail / (tile * ns)));
  char* out = ring + avail;
  const uint32_t NS = uint32_t(stages), K = uint32_t(kOutBufs);
  // does anybody wait for this channel's per-chunk signals?
  const bool need_signal = (reduce && !is_root) || a.exit_wait || ((t.children & ~t.leafmask) != 0u);
  unsigned int* ctr = t.ctr >= 0 ? reinterpret_cast<unsigned int*>(a.ctrl + 2) + t.ctr : nullptr;
  // A copy that signals every chunk drains its bulk stores (wait_group 0)
  // before the flag store, which stalls the next chunk's stores.  Split the
  // stage ring into two halves, chunks alternating between them, each drained
  // by its own store thread in its own warp (bulk groups are per thread; a
  // blocked wait stalls the whole warp): one half's drain overlaps the other
  // half's stores, and no signal is delayed.
  // Only when a chunk fits half the ring: longer chunks would leave the
  // other half idle (A/B: DGX-1V Broadcast 256 MiB, 4 MiB chunks, 30% slower).
  const bool short_chunks = !t.merged && (tr.chunk + tile - 1) / tile <= int64_t(NS / 2);
  const uint32_t R = (!reduce && need_signal && NS >= 2 && a.split_ring && short_chunks) ? 2u : 1u;
  const uint32_t H = NS / R;

  if (warp == 0) {
    // ------------------------------------------------ producer
    uint32_t gq[2] = {0u, 0u};  // tiles issued per sub-ring
    uint64_t p_acq = 0, p_issue = 0;  // trace stamps (written at the end)
    uint32_t nord = 0;          // chunks taken so far (sub-ring = nord % R)
    int cs = t.c0;  // static sequence
    // dynamic tasks: the first chunk is the CTA's own index (no atomic round
    // trip on the critical path); later chunks come from the counter, offset
    // by the number of CTAs.  When every CTA owns at most one chunk the
    // counter is never touched.
    const int nch = t.merged ? t.c1 : tr.nchunks;
    bool first_chunk = true;
    for (;;) {
      int c;
      if (ctr) {
        if (first_chunk && t.cta_idx >= 0) {  // a joining CTA (cta_idx -1) only uses the counter
          c = t.cta_idx;
          first_chunk = false;
        } else if (nch <= t.cta_cnt) {
          break;
        } else {
          unsigned int got = 0;
          if (lane == 0) got = atomicAdd(ctr, 1u);
          c = int(__shfl_sync(0xffffffffu, got, 0)) + t.cta_cnt;
        }
        if (c >= nch) break;
      } else {
        c = cs;
        cs += t.cstride;
        if (c >= t.c1) break;
      }
      if (sh.abort) break;
      const uint32_t wmask = reduce ? (t.children & ~t.leafmask) : (need_bflag ? 1u : 0u);
      const bool ok = wait_chunk_inputs(a, t, c, need_bflag, ctl);
      if (!ok) {
        if (lane == 0) sh.abort = 1;
        break;
      }
      if (lane == 0 && nord == 0) p_acq = stamp(a);
      int64_t b0, b1;
      if (t.merged) {  // one-hop roots over every rank: a chunk is a byte range
        b0 = int64_t(c) * a.mchunk;
        b1 = min(a.mbytes, b0 + a.mchunk);
      } else {
        b0 = tr.lo + int64_t(c) * tr.chunk;
        b1 = min(tr.hi, b0 + tr.chunk);
      }
      const int64_t body = ((b1 - b0) >> 4) << 4;
      if (body != b1 - b0) {  // sub-16-byte tail: scalar, by the producer warp
        if (reduce) {
          const int es = DT == BLINK_BFLOAT16 ? 2 : 4;
          for (int64_t off = b0 + body + int64_t(lane) * es; off < b1; off += 32 * es)
            Scalar<DT, OP>::reduce(sh.srcs, nsrc, sh.dsts, ndst, off, avg_m);
        } else {
          for (int64_t off = b0 + body + lane; off < b1; off += 32) {
            const char ch = __ldcg(sh.srcs[0] + off);
            for (int d = 0; d < ndst; ++d) sh.dsts[d][off] = ch;
          }
        }
        __syncwarp();
      }
      if (lane == 0) {
        if (wmask) fence_proxy_async();  // acquired flags order the TMA reads below
        if (c == t.c0 || (ctr && nord == 0)) p_issue = stamp(a);
        const uint32_t r = nord % R;
        uint32_t& g = gq[r];
        const int ntiles = body > 0 ? int((body + tile - 1) / tile) : 1;
        for (int k = 0; k < ntiles; ++k, ++g) {
          const uint32_t s = r * H + g % H;
          if (!mbar_wait_or_abort(&sh.empty[s], ((g / H) & 1u) ^ 1u, sh)) break;
          const int64_t off = int64_t(k) * tile;
          const uint32_t tb = uint32_t(max(int64_t(0), min(int64_t(tile), body - off)));
          TileMeta& mt = sh.smeta[s];
          mt.off = b0 + off;
          mt.c = c;
          mt.tb = int(tb);
          mt.last = k == ntiles - 1;
          if (tb == 0) {
            mbar_arrive(&sh.full[s]);  // empty tile (tail-only chunk): meta only
            continue;
          }
          mbar_expect_tx(&sh.full[s], tb * uint32_t(ns));
          char* st = ring + size_t(s) * tile * ns;
          if (a.l2_hint) {
            const uint64_t pol = l2_evict_first_policy();
            for (int j = 0; j < ns; ++j)
              tma_load_hint(st + size_t(j) * tile, sh.srcs[j] + b0 + off, tb, &sh.full[s], pol);
          } else {
            for (int j = 0; j < ns; ++j) tma_load(st + size_t(j) * tile, sh.srcs[j] + b0 + off, tb, &sh.full[s]);
          }
        }
      }
      __syncwarp();
      ++nord;
    }
    if (lane == 0) {
      trace_at(a, 8, p_acq);
      trace_at(a, 3, p_issue);
    }
    if (lane == 0)  // end of stream, in every sub-ring
      for (uint32_t r = 0; r < R; ++r) {
        const uint32_t s = r * H + gq[r] % H;
        if (mbar_wait_or_abort(&sh.empty[s], ((gq[r] / H) & 1u) ^ 1u, sh)) {
          sh.smeta[s].c = -1;
          mbar_arrive(&sh.full[s]);
        }
      }
  } else if (warp >= 1 && uint32_t(warp) <= R && lane == 0) {
    // ------------------------------------------------ store (warp 1 + r: sub-ring r)
    const uint32_t r = uint32_t(warp) - 1u;
    const int Dwant = a.store_depth >= 0 ? a.store_depth : 2;
    const int D = min(Dwant, (reduce ? int(K) : int(H)) - 1);
    auto release = [&](uint32_t gt) {
      if (reduce)
        mbar_arrive(&sh.oempty[gt % K]);
      else
        mbar_arrive(&sh.empty[r * H + gt % H]);
    };
    int kept = 0;
    uint64_t s_full = 0, s_store = 0, s_eos = 0;  // trace stamps (written at the end)
    bool first = true;
    // Deferred chunk signals (a5): a finished chunk is published once its
    // bulk-store group has completed, without draining the stores behind it.
    // Groups complete in order, so after wait_group<kSigDepth> every chunk
    // whose last group is at least kSigDepth groups old is complete.  When
    // the next tile is not ready yet the store thread drains instead (nothing
    // to overlap, and a deep tree's next hop waits on this signal).
    constexpr int kSigDepth = 3;
    constexpr int kPend = 8;
    int pend_c[kPend];
    uint32_t pend_g[kPend];
    int npend = 0;
    uint32_t groups = 0;  // bulk groups committed so far
    auto publish_upto = [&](uint32_t done_groups) {  // groups [0, done_groups) are complete
      int k = 0;
      while (k < npend && pend_g[k] <= done_groups) ++k;
      if (k == 0) return;
      fence_proxy_async();
      for (int q = 0; q < k; ++q) signal_chunk(a, t, pend_c[q], is_root, ctl);
      for (int q = k; q < npend; ++q) {
        pend_c[q - k] = pend_c[q];
        pend_g[q - k] = pend_g[q];
      }
      npend -= k;
    };
    for (uint32_t g = 0;; ++g) {
      TileMeta mt;
      const char* src;
      uint64_t* fb;
      uint32_t par;
      if (reduce) {
        const uint32_t o = g % K;
        fb = &sh.ofull[o];
        par = (g / K) & 1u;
        src = out + size_t(o) * tile;
      } else {
        const uint32_t s = r * H + g % H;
        fb = &sh.full[s];
        par = (g / H) & 1u;
        src = ring + size_t(s) * tile;
      }
      if (npend > 0 && !mbar_test(fb, par)) {  // idle: publish everything now
        tma_wait_all();
        for (int j = kept - 1; j >= 0; --j) release(g - 1u - uint32_t(j));
        kept = 0;
        publish_upto(groups);
      }
      if (!mbar_wait_or_abort(fb, par, sh)) break;
      mt = reduce ? sh.ometa[g % K] : sh.smeta[r * H + g % H];
      if (g == 0) s_full = stamp(a);
      if (mt.c < 0) {
        s_eos = stamp(a);
        break;
      }
      if (a.l2_hint) {
        const uint64_t pol = l2_evict_first_policy();
        for (int d = 0; d < ndst && mt.tb > 0; ++d) tma_store_hint(sh.dsts[d] + mt.off, src, uint32_t(mt.tb), pol);
      } else {
        for (int d = 0; d < ndst && mt.tb > 0; ++d) tma_store(sh.dsts[d] + mt.off, src, uint32_t(mt.tb));
      }
      tma_commit();
      ++groups;
      if (first) {
        s_store = stamp(a);
        first = false;
      }
      if (++kept > D) {
        if (D >= 2)
          tma_wait_read<2>();
        else if (D == 1)
          tma_wait_read<1>();
        else
          tma_wait_read<0>();
        release(g - uint32_t(D));
        --kept;
      }
      if (need_signal) {
        if (mt.last) {
          if (npend == kPend) {  // full: drain the oldest first
            tma_wait_all();
            publish_upto(groups);
          }
          pend_c[npend] = mt.c;
          pend_g[npend] = groups;
          ++npend;
        }
        if (npend > 0 && !a.defer_signal) {  // BLINK_DEFER_SIGNAL=0: drain per chunk
          tma_wait_all();
          publish_upto(groups);
        } else if (npend > 0 && groups >= uint32_t(kSigDepth) && pend_g[0] <= groups - kSigDepth) {
          tma_wait_group<kSigDepth>();
          publish_upto(groups - kSigDepth);
        }
      }
    }
    tma_wait_all();
    const uint64_t s_drained = stamp(a);
    fence_proxy_async();
    if (npend > 0) publish_upto(groups);
    const uint64_t s_pub = stamp(a);
    if (r == 0) {
      trace_at(a, 4, s_store);
      trace_at(a, 9, s_full);
      trace_at(a, 10, s_eos);
      trace_at(a, 11, s_drained);
      trace_at(a, 12, s_pub);
      trace_at(a, 5, s_pub);
    }
  } else if (reduce && warp >= 2) {
    // ------------------------------------------------ consumers
    const int ct = threadIdx.x - 64, CT = ncons * 32;
    const int vstride = tile >> 4;
    for (uint32_t g = 0;; ++g) {
      const uint32_t s = g % NS, o = g % K;
      if (!mbar_wait_or_abort(&sh.full[s], (g / NS) & 1u, sh)) break;
      const TileMeta mt = sh.smeta[s];
      if (!mbar_wait_or_abort(&sh.oempty[o], ((g / K) & 1u) ^ 1u, sh)) break;
      if (mt.c >= 0) {
        const int vecs = mt.tb >> 4;
        const uint4* st = reinterpret_cast<const uint4*>(ring + size_t(s) * tile * ns);
        uint4* ob = reinterpret_cast<uint4*>(out + size_t(o) * tile);
        for (int vv = ct; vv < vecs; vv += CT) {
          Acc<DT> acc;
          widen<DT>(acc, st[vv]);
          for (int j = 1; j < nsrc; ++j) combine<DT, OP>(acc, st[j * vstride + vv]);
          if (OP == BLINK_AVG && avg_m) divide<DT>(acc, avg_m);
          ob[vv] = narrow<DT>(acc);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      if (ct == 0) sh.ometa[o] = mt;
      __syncwarp();
      if (lane == 0) {
        if (mt.c >= 0) mbar_arrive(&sh.empty[s]);
        mbar_arrive(&sh.ofull[o]);
      }
      if (mt.c < 0) break;
    }
  }
  __syncthreads();
}

// Register/LSU path (misaligned buffers, BLINK_TMA=0): all threads per chunk.
template <int DT, int OP, bool VEC>
__device__ void run_lsu(const LaunchArgs& a, const DevTask& t, const DevTree& tr, bool is_root,
                        bool need_bflag, Shared& sh, const Ctl& ctl) {
  for (int c = t.c0; c < t.c1; c += t.cstride) {
    if (threadIdx.x < 32) {
      const bool ok = wait_chunk_inputs(a, t, c, need_bflag, ctl);
      if (threadIdx.x == 0) sh.ok = ok;
    }
    __syncthreads();
    const bool ok = sh.ok;
    if (ok) {
      int64_t b0 = tr.lo + int64_t(c) * tr.chunk;
      int64_t b1 = min(tr.hi, b0 + tr.chunk);
      if (t.merged) {  // one-hop roots over every rank: a chunk is a byte range
        b0 = int64_t(c) * a.mchunk;
        b1 = min(a.mbytes, b0 + a.mchunk);
      }
      if (t.role == kRoleReduce)
        reduce_range<DT, OP, VEC>(sh.srcs, sh.nsrc, sh.dsts, sh.ndst, b0, b1,
                                  (OP == BLINK_AVG && is_root) ? a.nranks : 0);
      else
        copy_range<VEC>(sh.srcs[0], sh.dsts, sh.ndst, b0, b1);
    }
    __syncthreads();  // every thread's stores of chunk c are issued (and sh.ok read)
    if (!ok) break;
    // merged channels exist only in single launches of independent roots:
    // nobody waits for their per-chunk signals
    if (threadIdx.x == 0 && !t.merged) signal_chunk(a, t, c, is_root, ctl);
  }
}

template <int DT, int OP, bool VEC>
__global__ void __launch_bounds__(256, 1) exec_kernel(const LaunchArgs a_in) {
  __shared__ Shared sh;
  __shared__ uint64_t s_epoch;
  extern __shared__ __align__(128) char s_ring[];
  // Epoch = launches completed on this device group + 1, read from device
  // memory so that CUDA-graph replays get fresh epochs.
  const LaunchArgs& a = a_in;
  DevTask t0;
  if (a.merged_all) {  // one merged channel: the task differs only by index
    t0 = a.mtask;
    t0.cta_idx = blockIdx.x;
    t0.c0 = blockIdx.x;
  } else {
    t0 = a.tasks[blockIdx.x];
  }
  // A merged single launch (one-hop AllReduce roots, every rank in this
  // launch) reads and writes no flag: it needs no epoch, and its last CTA just
  // advances the counter -- no dependent load before the first TMA load.
  const bool no_flags = a.merged_all && !a.exit_wait;
  // Programmatic dependent launch: everything above reads only kernel
  // parameters and the host-written task table; every access to memory the
  // previous kernel in the stream may touch (epoch, counters, flags, user
  // buffers, trace) comes after this wait.  A no-op without the attribute.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    if (a.trace)
      for (int k = 1; k < kTraceSlots; ++k) a.trace[size_t(blockIdx.x) * kTraceSlots + k] = 0;
    trace(a, 0);
    s_epoch = no_flags ? 0 : *reinterpret_cast<volatile uint64_t*>(a.ctrl) + 1;
    trace(a, 1);
  }
  __syncthreads();
  const int v = t0.rank;
  const Ctl ctl{s_epoch, a.timeout_ns, a.err, a.scope_sys != 0};
  uint64_t* myflags = a.flags[v];
  const bool ws = VEC && a.use_tma && blockDim.x >= 128;

  // entry: my send is ready and my recv may be overwritten (epoch e).  Every
  // segment of this CTA publishes its entry before any segment waits.
  if (threadIdx.x == 0 && a.exit_wait) {
    bool fenced = false;
    for (int ti = blockIdx.x; ti >= 0; ti = a.tasks[ti].next) {
      const DevTask& tt = a.tasks[ti];
      if (!tt.do_entry) continue;
      // earlier kernels' writes to send are ordered by the launch boundary;
      // across devices / processes publish with a release fence anyway
      if (!fenced && ctl.sys) fence_release(true);
      fenced = true;
      for (int u = 0; u < a.nranks; ++u)
        if (u != tt.rank) st_relaxed(a.flags[u] + entry_idx(tt.rank), ctl.epoch, ctl.sys);
    }
  }

  // segments: usually one; packed launches chain contiguous chunk ranges of
  // independent channels so that every SM carries the same number of bytes
  // Then work stealing (a6, TMA path, dynamic channels): a CTA whose own
  // channel has handed out every chunk joins the channel of this launch with
  // the most chunks not yet taken and takes chunks from its counter,
  // until no channel has any left.  Channels still hand out chunks in
  // increasing order and a joined chunk's inputs come from chunks that other
  // resident CTAs hold or will take, so DESIGN 2b's deadlock argument stands.
  __shared__ int s_join;
  bool stealing = false;
  for (int ti = blockIdx.x;;) {
    DevTask t;
    if (!stealing) {
      if (ti < 0) {
        if (!(ws && a.nchan > 0)) break;
        stealing = true;
        continue;
      }
      t = ti == int(blockIdx.x) ? t0 : a.tasks[ti];
      ti = t.next;
    } else {
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const volatile unsigned int* ctrs = reinterpret_cast<const volatile unsigned int*>(a.ctrl + 2);
        int best = -1, brem = 1;
        for (int ci = lane; ci < a.nchan; ci += 32) {
          const DevTask& r = a.tasks[a.chan0 + ci];
          const int rem = r.tr.nchunks - r.cta_cnt - int(ctrs[r.ctr]);
          // only where the channel's own CTAs still have > 2 rounds of
          // chunks: a joiner's set-up costs about one chunk, and at the tail
          // of small calls joiners only add pollers (A/B: 1 MiB 1 us slower)
          if (rem > 2 * r.cta_cnt && rem > brem) {
            brem = rem;
            best = ci;
          }
        }
        for (int o = 16; o > 0; o >>= 1) {  // most chunks left; ties: lowest channel
          const int orem = __shfl_xor_sync(0xffffffffu, brem, o);
          const int ob = __shfl_xor_sync(0xffffffffu, best, o);
          if (orem > brem || (orem == brem && ob >= 0 && (best < 0 || ob < best))) {
            brem = orem;
            best = ob;
          }
        }
        if (lane == 0) s_join = best;
      }
      __syncthreads();
      const int j = s_join;
      if (j < 0) break;
      t = a.tasks[a.chan0 + j];
    }
    if (t.role != kRoleReduce && t.role != kRoleBcast) continue;
    const int w = t.rank;
    uint64_t* wflags = a.flags[w];
    const DevTree tr = t.tr;
    const bool is_root = t.parent < 0;
    // entry handshake (warp 0): leaf children's send is ready once they
    // entered; Broadcast / AllGather push into children's recv only after they
    // entered
    bool entry_ok = true;
    if (threadIdx.x < 32) {
      const bool pushes = is_push_coll(a.coll);
      // one launch holding every rank: all inputs are final at launch and all
      // outputs free, so there is nothing to hand shake
      const uint32_t emask = !a.exit_wait ? 0u
                             : (t.role == kRoleReduce ? t.leafmask : (pushes ? t.children : 0u));
      entry_ok = warp_wait(emask, [&](int u) { return wflags + entry_idx(u); }, ctl);
    }
    if (threadIdx.x < 32) {
      // warp 0 builds the operand / destination lists: lane u looks at rank u
      // (parallel parameter loads instead of one thread walking the ranks);
      // sources in ascending rank order (R#12), destinations in rank order
      const int u = threadIdx.x;
      const uint32_t me = 1u << w;
      bool is_src = false, from_send = false, is_dst = false;
      char* su = nullptr;
      char* ru = nullptr;
      if (u < a.nranks) {
        su = a.send[u];
        ru = a.recv[u];
        const uint32_t bit = 1u << u;
        if (t.role == kRoleReduce) {
          is_src = ((t.children | me) & bit) != 0u;
          from_send = ((t.leafmask | me) & bit) != 0u;
          // ReduceScatter keeps the result at the root
          is_dst = u == w || (is_root && a.coll == kAllReduce && (t.children & bit));
          // link-graph ReduceScatter: partials of inner ranks live in the relay
          // area (an internal child's source, a non-root's destination)
          if (a.relay[u] && !(u == w && is_root)) ru = a.relay[u];
        } else {
          const bool src_root = is_push_coll(a.coll) && is_root;
          is_src = u == w;
          from_send = src_root;
          // the root's own copy (Gather: only the gather root holds a recv)
          is_dst = (t.children & bit) != 0u ||
                   (u == w && src_root && su != ru && (a.coll != kGather || w == a.bcast_root));
        }
      }
      const uint32_t below = (1u << u) - 1u;
      const uint32_t sm = __ballot_sync(0xffffffffu, is_src), dm = __ballot_sync(0xffffffffu, is_dst);
      if (is_src) sh.srcs[__popc(sm & below)] = from_send ? su : ru;
      if (is_dst) sh.dsts[__popc(dm & below)] = ru;
      if (u == 0) {
        sh.nsrc = __popc(sm);
        sh.ndst = __popc(dm);
        sh.abort = entry_ok ? 0 : 1;
        if (ws) {  // (re)initialise the ring's barriers: every segment starts drained
          const uint32_t ncw = t.role == kRoleReduce ? (blockDim.x >> 5) - 2 : 1;
          for (int k = 0; k < kMaxStages; ++k) {
            mbar_init(&sh.full[k], 1);
            mbar_init(&sh.empty[k], ncw);
          }
          for (int k = 0; k < kOutBufs; ++k) {
            mbar_init(&sh.ofull[k], ncw);
            mbar_init(&sh.oempty[k], 1);
          }
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) trace(a, 2);
    const bool need_bflag = (t.role == kRoleBcast) && !(is_push_coll(a.coll) && is_root);
    const bool aborted = sh.abort;
    if (!aborted) {
      if (ws)
        run_ws<DT, OP>(a, t, tr, is_root, need_bflag, sh, s_ring, ctl);
      else
        run_lsu<DT, OP, VEC>(a, t, tr, is_root, need_bflag, sh, ctl);
    }
    __syncthreads();  // segment drained; smem (lists, barriers) may be reused
    if (aborted) break;
  }
  const DevTask& t = t0;

  // exit: every final chunk of every tree not rooted here has arrived, which
  // also means every peer finished reading this rank's buffers (causality).
  if (a.exit_wait) {
    __syncthreads();
    // the (tree, chunk) flags of this rank, flattened; this thread waits for
    // items g, g + G, ... (walking the trees once, not every item)
    const int G = t.exit_cnt * int(blockDim.x);
    int k = t.exit_idx * int(blockDim.x) + int(threadIdx.x);
    int base = 0;
    for (int i = 0; i < a.ntrees; ++i) {
      const DevTree& tr = a.ptrees[i];
      if (tr.root == v || !((tr.members >> v) & 1u)) continue;
      for (; k < base + tr.nchunks; k += G) wait_ge(myflags + bflag_idx(i, k - base), ctl);
      base += tr.nchunks;
    }
    fence_acquire(ctl.sys);
  }
  // the last CTA to finish advances the device epoch for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    trace(a, 6);
    // the next launch is stream-ordered after this one: no fences needed here
    const unsigned long long prev = atomicAdd(reinterpret_cast<unsigned long long*>(a.ctrl + 1), 1ull);
    if (prev + 1 == gridDim.x) {
      a.ctrl[1] = 0;
      for (int k = 0; k < a.nctr; ++k) reinterpret_cast<unsigned int*>(a.ctrl + 2)[k] = 0u;
      if (no_flags)  // = ctrl[0] + 1, the epoch this launch would have read
        atomicAdd(reinterpret_cast<unsigned long long*>(a.ctrl), 1ull);
      else
        atomicExch(reinterpret_cast<unsigned long long*>(a.ctrl), (unsigned long long)ctl.epoch);
    }
    trace(a, 7);
  }
}

template <bool VEC>
__global__ void copy_kernel(char* dst, const char* src, int64_t bytes) {
  const int64_t T = int64_t(gridDim.x) * blockDim.x;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t vb = 0;
  if (VEC) {
    const int64_t nv = bytes >> 4;
    for (int64_t j = tid; j < nv; j += T)
      __stcg(reinterpret_cast<uint4*>(dst) + j, __ldcg(reinterpret_cast<const uint4*>(src) + j));
    vb = nv << 4;
  }
  for (int64_t j = vb + tid; j < bytes; j += T) dst[j] = src[j];
}

// ------------------------------------------------------------------ LL protocol
// Small calls on switch plans (blink_internal.h "LL protocol").  Lines are
// two u64 words {data32 | flag << 32}: each word is single-copy atomic, so a
// word whose flag equals the call's epoch carries that call's data.
__device__ __forceinline__ void ll_store(uint4* p, uint2 d, uint32_t f) {
  const uint64_t w0 = uint64_t(d.x) | (uint64_t(f) << 32), w1 = uint64_t(d.y) | (uint64_t(f) << 32);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
// 8 payload bytes of a user buffer; `valid` (a multiple of the element size)
// bytes are read, the rest is zero.  Buffers are element-aligned.
__device__ __forceinline__ uint2 ld8(const char* p, int valid) {
  if (valid == 8 && (reinterpret_cast<uintptr_t>(p) & 7) == 0) return __ldcg(reinterpret_cast<const uint2*>(p));
  uint2 r = make_uint2(0u, 0u);
  unsigned short* h = reinterpret_cast<unsigned short*>(&r);
  for (int b = 0; b < valid; b += 2) h[b >> 1] = __ldcg(reinterpret_cast<const unsigned short*>(p + b));
  return r;
}
__device__ __forceinline__ void st8(char* p, uint2 v, int valid) {
  if (valid == 8 && (reinterpret_cast<uintptr_t>(p) & 7) == 0) {
    *reinterpret_cast<uint2*>(p) = v;
    return;
  }
  const unsigned short* h = reinterpret_cast<const unsigned short*>(&v);
  for (int b = 0; b < valid; b += 2) *reinterpret_cast<unsigned short*>(p + b) = h[b >> 1];
}
// Combine of 8-byte payloads with the executor's arithmetic (R#12, R#13):
// fp32 accumulation, RNE, no FMA; bf16 widened exactly and rounded once.
template <int DT, int OP>
struct Acc8 {
  static constexpr int N = DT == BLINK_BFLOAT16 ? 4 : 2;
  float f[N];
  int i[N];
  __device__ __forceinline__ void unpack(uint2 x, float* g, int* j) const {
    if constexpr (DT == BLINK_BFLOAT16) {
      g[0] = bf_lo(x.x); g[1] = bf_hi(x.x); g[2] = bf_lo(x.y); g[3] = bf_hi(x.y);
    } else if constexpr (DT == BLINK_FLOAT32) {
      g[0] = __uint_as_float(x.x); g[1] = __uint_as_float(x.y);
    } else {
      j[0] = int(x.x); j[1] = int(x.y);
    }
  }
  __device__ __forceinline__ void init(uint2 x) { unpack(x, f, i); }
  __device__ __forceinline__ void add(uint2 x) {
    float g[N];
    int j[N];
    unpack(x, g, j);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if constexpr (DT == BLINK_INT32)
        i[k] = iop<OP>(i[k], j[k]);
      else
        f[k] = fop<OP>(f[k], g[k]);
    }
  }
  __device__ __forceinline__ void divide(int m) {  // AVG at the root (R#28)
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if constexpr (DT == BLINK_INT32)
        i[k] = avg_div(i[k], m);
      else
        f[k] = avg_div(f[k], m);
    }
  }
  __device__ __forceinline__ uint2 out() const {
    if constexpr (DT == BLINK_BFLOAT16)
      return make_uint2(f2bf(f[0]) | (f2bf(f[1]) << 16), f2bf(f[2]) | (f2bf(f[3]) << 16));
    else if constexpr (DT == BLINK_FLOAT32)
      return make_uint2(__float_as_uint(f[0]), __float_as_uint(f[1]));
    else
      return make_uint2(unsigned(i[0]), unsigned(i[1]));
  }
};

__device__ __forceinline__ void ll_trace(const LLArgs& a, int slot) {
  if (a.trace) a.trace[size_t(blockIdx.x) * kTraceSlots + slot] = globaltimer();
}

// Batched poll: the lines ptr(u) of every u < U with bit u of `act` set are
// loaded back to back, then only the ones whose flags are not yet `f` are
// reloaded, so a thread's round trips overlap.  d[u] gets line u's payload.
// (Unrolled with compile-time indices: no local-memory arrays.)  False on
// timeout / abort.
template <int U, class P>
__device__ __forceinline__ bool ll_poll_n(P ptr, uint32_t act, uint32_t f, uint2* d, const LLArgs& a) {
  uint64_t w0[U], w1[U];
  bool done[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    done[u] = !((act >> u) & 1u);
    if (!done[u])
      asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0[u]), "=l"(w1[u]) : "l"(ptr(u)) : "memory");
  }
  uint64_t t0 = 0;
  for (int spin = 0;; ++spin) {
    bool all = true;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (done[u]) continue;
      if (uint32_t(w0[u] >> 32) == f && uint32_t(w1[u] >> 32) == f) {
        d[u] = make_uint2(uint32_t(w0[u]), uint32_t(w1[u]));
        done[u] = true;
      } else {
        all = false;
      }
    }
    if (all) return true;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (!done[u])
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0[u]), "=l"(w1[u]) : "l"(ptr(u)) : "memory");
    if ((spin & 255) == 255) {
      if (ld_volatile_int(a.err) != 0) return false;
      const uint64_t now = globaltimer();
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > a.timeout_ns) {
        *reinterpret_cast<volatile int*>(a.err) = int(BLINK_ERR_TIMEOUT);
        return false;
      }
    }
  }
}

// One launch runs ranks a.ranks[0 .. nlocal), a.ctas_per_rank CTAs each.
// AllReduce on m one-hop trees (tree j rooted at j owns slice j):
//   P1 (leaf)  push my send slice j into root j's IN[p][me], every j != me;
//   P2 (root)  for my slice: poll IN[p][u] of every leaf u, combine with my
//              send in ascending rank order, write my recv and push the
//              result into OUT[p][me] of every leaf;
//   P3 (leaf)  poll my OUT[p][j] for every j != me and write my recv.
// Broadcast (one-hop star): the root pushes its send into every other rank's
// OUT[p] run; the others poll and copy out.  Every thread runs its P1 share
// before any wait, so progress needs only that every CTA eventually runs.
// Work items are (slice, line) pairs spread over all threads of the rank, and
// each thread issues the loads of up to kLLU items (or, in P2, of all m
// operands of a line) before waiting on any of them: a phase costs about one
// round trip, not one per peer.
constexpr int kLLU = 4;
template <int DT, int OP>
__global__ void __launch_bounds__(kLLThreads) ll_kernel(const LLArgs a) {
  const int v = a.ranks[blockIdx.x / a.ctas_per_rank];
  const int cta = blockIdx.x % a.ctas_per_rank;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: see exec_kernel
  if (threadIdx.x == 0 && a.trace)  // slots this kernel does not stamp read 0
    for (int k = 1; k < kTraceSlots; ++k) a.trace[size_t(blockIdx.x) * kTraceSlots + k] = 0;
  if (threadIdx.x == 0) ll_trace(a, 0);
  const int m = a.nranks;
  const int64_t T = int64_t(a.ctas_per_rank) * blockDim.x;
  const int64_t t0 = int64_t(cta) * blockDim.x + threadIdx.x;
  const size_t cap = size_t(a.cap);
  // every thread reads the epoch (one broadcast load; no block barrier); the
  // CTA's finish counter is bumped only after __syncthreads below
  const uint64_t e = *reinterpret_cast<volatile uint64_t*>(a.ctrl) + 1;
  const uint32_t f = uint32_t(e);
  const size_t p = size_t(e & 1u);
  uint4* const my = a.ll[v];
  // Ranks in other launches (per-rank launches, processes): publish entry(e)
  // -- this rank finished call e-1, so it no longer reads the LL lines of
  // parity p^1 -- in every peer's flag words (they precede the LL area).  A
  // Broadcast root waits for every leaf's entry(e-1) before it overwrites
  // their parity-p lines: nothing else stops a root that only pushes from
  // running two calls ahead of a leaf (AllReduce results depend on every
  // rank's previous call, so its roots cannot).
  const bool multi = a.nlocal < m;
  auto flags_of = [&](int u) {
    return reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(a.ll[u]) - kFlagBytes);
  };
  if (multi && cta == 0 && threadIdx.x < m && int(threadIdx.x) != v)
    st_relaxed(flags_of(threadIdx.x) + entry_idx(v), e, a.scope_sys != 0);
  __shared__ int s_root_ok;
  if (multi && a.coll == kBroadcast && v == a.root) {
    if (threadIdx.x < 32) {
      const Ctl ctl{e - 1, a.timeout_ns, a.err, a.scope_sys != 0};
      const uint32_t leaves = ((m >= 32 ? 0u : (1u << m)) - 1u) & ~(1u << v);
      const bool ok = warp_wait(leaves, [&](int u) { return flags_of(v) + entry_idx(u); }, ctl);
      if (threadIdx.x == 0) s_root_ok = ok;  // timeout: error word set, no pushes
    }
    __syncthreads();
  }
  auto in_area = [&](uint4* base, int src) { return base + (p * m + src) * cap; };
  auto out_area = [&](uint4* base, int j) { return base + ((2 + p) * m + j) * cap; };
  bool ok = true;
  // rank v: poll its OUT[p][0] lines (the final value from its parent),
  // write them to recv and forward them to its children's OUT[p][0]
  auto tree_down = [&](uint32_t kids) {
    const int64_t len = a.bytes, nl = (len + 7) >> 3;
    const uint4* src = out_area(my, 0);
    for (int64_t k0 = t0; k0 < nl; k0 += kLLU * T) {
      uint2 d[kLLU];
      uint32_t act = 0;
#pragma unroll
      for (int u = 0; u < kLLU; ++u)
        if (k0 + u * T < nl) act |= 1u << u;
      if (!ll_poll_n<kLLU>([&](int u) { return src + k0 + u * T; }, act, f, d, a)) return false;
#pragma unroll
      for (int u = 0; u < kLLU; ++u)
        if ((act >> u) & 1u) {
          const int64_t k = k0 + u * T;
          st8(a.recv[v] + 8 * k, d[u], int(min(int64_t(8), len - 8 * k)));
          for (int c = 0; c < m; ++c)
            if ((kids >> c) & 1u) ll_store(out_area(a.ll[c], 0) + k, d[u], f);
        }
    }
    return true;
  };
  if (a.tree) {
    // One multi-level tree (R#27): child u's partial lines go to its
    // parent's IN[p][u]; final lines travel down through OUT[p][0].  Every
    // node combines {own send} + children in ascending rank order with the
    // executor's arithmetic (one rounding per node, R#12/R#13), like the
    // tree executor and the oracle.
    const int rt = a.tree_root;
    uint32_t kids = 0;
    for (int u = 0; u < m; ++u)
      if (a.parent[u] == v) kids |= 1u << u;
    const int64_t len = a.bytes, nl = (len + 7) >> 3;
    if (a.coll == kAllReduce) {
      for (int64_t k = t0; k < nl; k += T) {
        const int valid = int(min(int64_t(8), len - 8 * k));
        const uint2 own = ld8(a.send[v] + 8 * k, valid);
        uint2 d[kMaxRanks];
        if (kids && !ll_poll_n<kMaxRanks>([&](int u) { return in_area(my, u) + k; }, kids, f, d, a)) {
          ok = false;
          break;
        }
        Acc8<DT, OP> acc;
        bool first = true;
#pragma unroll
        for (int u = 0; u < kMaxRanks; ++u) {
          if (u >= m) break;
          if (u != v && !((kids >> u) & 1u)) continue;
          const uint2 x = u == v ? own : d[u];
          if (first)
            acc.init(x);
          else
            acc.add(x);
          first = false;
        }
        if (OP == BLINK_AVG && v == rt) acc.divide(m);
        const uint2 r = acc.out();
        if (v == rt) {
          st8(a.recv[v] + 8 * k, r, valid);
          for (int c = 0; c < m; ++c)
            if ((kids >> c) & 1u) ll_store(out_area(a.ll[c], 0) + k, r, f);
        } else {
          ll_store(in_area(a.ll[a.parent[v]], v) + k, r, f);
        }
      }
      if (ok && v != rt) ok = tree_down(kids);
    } else if (v == rt) {  // Broadcast root
      const int64_t kend = (multi && !s_root_ok) ? 0 : nl;
      for (int64_t k = t0; k < kend; k += T) {
        const int valid = int(min(int64_t(8), len - 8 * k));
        const uint2 x = ld8(a.send[v] + 8 * k, valid);
        if (a.recv[v] != a.send[v]) st8(a.recv[v] + 8 * k, x, valid);
        for (int c = 0; c < m; ++c)
          if ((kids >> c) & 1u) ll_store(out_area(a.ll[c], 0) + k, x, f);
      }
    } else {
      ok = tree_down(kids);
    }
  } else if (a.coll == kAllReduce) {
    int64_t lmax = 0;
    for (int j = 0; j < m; ++j) lmax = max(lmax, a.lo[j + 1] - a.lo[j]);
    const int64_t nlmax = (lmax + 7) >> 3;
    const int64_t tot = int64_t(m - 1) * nlmax;  // (slice j != v, line k) items
    auto item = [&](int64_t i, int& j, int64_t& k, int& valid) {
      const int jj = int(i / nlmax);
      k = i - int64_t(jj) * nlmax;
      j = jj + (jj >= v ? 1 : 0);
      const int64_t len = a.lo[j + 1] - a.lo[j];
      valid = int(min(int64_t(8), len - 8 * k));
      return i < tot && 8 * k < len;
    };
    // P1
    for (int64_t i0 = t0; i0 < tot; i0 += kLLU * T) {
      uint2 x[kLLU];
      int jv[kLLU];
      int64_t kv[kLLU];
      bool act[kLLU];
#pragma unroll
      for (int u = 0; u < kLLU; ++u) {
        int valid;
        act[u] = item(i0 + u * T, jv[u], kv[u], valid);
        if (act[u]) x[u] = ld8(a.send[v] + a.lo[jv[u]] + 8 * kv[u], valid);
      }
#pragma unroll
      for (int u = 0; u < kLLU; ++u)
        if (act[u]) ll_store(in_area(a.ll[jv[u]], v) + kv[u], x[u], f);
    }
    if (threadIdx.x == 0) ll_trace(a, 2);
    {  // P2
      const int64_t lo = a.lo[v], len = a.lo[v + 1] - lo, nl = (len + 7) >> 3;
      const uint32_t leaves = ((m >= 32 ? 0u : (1u << m)) - 1u) & ~(1u << v);
      for (int64_t k = t0; k < nl; k += T) {
        const int valid = int(min(int64_t(8), len - 8 * k));
        const uint2 own = ld8(a.send[v] + lo + 8 * k, valid);
        uint2 d[kMaxRanks];
        if (!ll_poll_n<kMaxRanks>([&](int u) { return in_area(my, u) + k; }, leaves, f, d, a)) {
          ok = false;
          break;
        }
        Acc8<DT, OP> acc;
#pragma unroll
        for (int u = 0; u < kMaxRanks; ++u) {
          if (u >= m) break;
          const uint2 x = u == v ? own : d[u];
          if (u == 0)
            acc.init(x);
          else
            acc.add(x);
        }
        if (OP == BLINK_AVG) acc.divide(m);
        const uint2 r = acc.out();
        st8(a.recv[v] + lo + 8 * k, r, valid);
        for (int u = 0; u < m; ++u)
          if (u != v) ll_store(out_area(a.ll[u], v) + k, r, f);
      }
    }
    if (threadIdx.x == 0) ll_trace(a, 3);
    // P3
    for (int64_t i0 = t0; i0 < tot && ok; i0 += kLLU * T) {
      const uint4* ps[kLLU];
      char* dst[kLLU];
      int val[kLLU];
      uint2 d[kLLU];
      uint32_t act = 0;
#pragma unroll
      for (int u = 0; u < kLLU; ++u) {
        int j, valid;
        int64_t k;
        ps[u] = nullptr;
        dst[u] = nullptr;
        val[u] = 0;
        if (item(i0 + u * T, j, k, valid)) {
          ps[u] = out_area(my, j) + k;
          dst[u] = a.recv[v] + a.lo[j] + 8 * k;
          val[u] = valid;
          act |= 1u << u;
        }
      }
      if (!ll_poll_n<kLLU>([&](int u) { return ps[u]; }, act, f, d, a)) {
        ok = false;
        break;
      }
#pragma unroll
      for (int u = 0; u < kLLU; ++u)
        if ((act >> u) & 1u) st8(dst[u], d[u], val[u]);
    }
  } else {  // Broadcast, one-hop star
    const int r = a.root;
    const int64_t len = a.bytes, nl = (len + 7) >> 3;
    if (v == r) {
      const int64_t kend = (multi && !s_root_ok) ? 0 : nl;
      for (int64_t k = t0; k < kend; k += T) {
        const int valid = int(min(int64_t(8), len - 8 * k));
        const uint2 x = ld8(a.send[r] + 8 * k, valid);
        if (a.recv[r] != a.send[r]) st8(a.recv[r] + 8 * k, x, valid);
        for (int u = 0; u < m; ++u)
          if (u != r) ll_store(out_area(a.ll[u], 0) + k, x, f);
      }
    } else {
      const uint4* src = out_area(my, 0);
      for (int64_t k0 = t0; k0 < nl; k0 += kLLU * T) {
        uint2 d[kLLU];
        uint32_t act = 0;
#pragma unroll
        for (int u = 0; u < kLLU; ++u)
          if (k0 + u * T < nl) act |= 1u << u;
        if (!ll_poll_n<kLLU>([&](int u) { return src + k0 + u * T; }, act, f, d, a)) break;
#pragma unroll
        for (int u = 0; u < kLLU; ++u)
          if ((act >> u) & 1u) {
            const int64_t k = k0 + u * T;
            st8(a.recv[v] + 8 * k, d[u], int(min(int64_t(8), len - 8 * k)));
          }
      }
    }
  }
  // the last CTA to finish advances the device epoch for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    ll_trace(a, 6);
    const unsigned long long prev = atomicAdd(reinterpret_cast<unsigned long long*>(a.ctrl + 1), 1ull);
    if (prev + 1 == gridDim.x) {
      a.ctrl[1] = 0;
      atomicExch(reinterpret_cast<unsigned long long*>(a.ctrl), (unsigned long long)e);
    }
    ll_trace(a, 7);
  }
}

typedef void (*ExecFn)(const LaunchArgs);

// Launch attributes: cooperative (co-residency checked by the driver) and/or
// programmatic stream serialization (PDL: the launch overlaps the previous
// kernel's tail; the kernels wait with griddepcontrol.wait before touching
// memory).  Eager launches gain from PDL only without the cooperative
// attribute (scripts/pdl_probe.cu), so the runtime sets one or the other.
void set_launch_attrs(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attr, bool cooperative, bool pdl) {
  int n = 0;
  if (cooperative) {
    attr[n].id = cudaLaunchAttributeCooperative;
    attr[n].val.cooperative = 1;
    ++n;
  }
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
}

template <int DT, bool VEC>
ExecFn pick_op(int op) {
  switch (op) {
    case BLINK_SUM: return exec_kernel<DT, BLINK_SUM, VEC>;
    case BLINK_PROD: return exec_kernel<DT, BLINK_PROD, VEC>;
    case BLINK_MIN: return exec_kernel<DT, BLINK_MIN, VEC>;
    case BLINK_MAX: return exec_kernel<DT, BLINK_MAX, VEC>;
    case BLINK_AVG: return exec_kernel<DT, BLINK_AVG, VEC>;
  }
  return nullptr;
}

ExecFn pick(int coll, int dtype, int op, bool vec) {
  if (is_push_coll(coll)) return vec ? exec_kernel<BLINK_FLOAT32, BLINK_SUM, true>
                                     : exec_kernel<BLINK_FLOAT32, BLINK_SUM, false>;
  switch (dtype) {
    case BLINK_FLOAT32: return vec ? pick_op<BLINK_FLOAT32, true>(op) : pick_op<BLINK_FLOAT32, false>(op);
    case BLINK_BFLOAT16: return vec ? pick_op<BLINK_BFLOAT16, true>(op) : pick_op<BLINK_BFLOAT16, false>(op);
    case BLINK_INT32: return vec ? pick_op<BLINK_INT32, true>(op) : pick_op<BLINK_INT32, false>(op);
  }
  return nullptr;
}

}  // namespace

cudaError_t launch_exec(const LaunchArgs& a, int grid, int threads, bool vec, void* stream,
                        bool cooperative, bool pdl) {
  ExecFn fn = pick(a.coll, a.dtype, a.op, vec);
  if (!fn) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = vec ? a.smem_bytes : 0;
  // cudaFuncSetAttribute is per device: remember it per (device, kernel)
  constexpr int kDevs = 64;
  static bool attr_set[kDevs][5][3][5][2] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevs) dev = -1;
  bool unknown_dev = false;
  bool& done = dev >= 0 ? attr_set[dev][a.coll][a.dtype][a.op][vec] : unknown_dev;
  if (!done) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         vec ? kMaxSmemBytes : 0);
    if (e != cudaSuccess) return e;
    done = true;
  }
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  set_launch_attrs(cfg, attr, cooperative, pdl);
  return cudaLaunchKernelEx(&cfg, fn, a);
}

typedef void (*LLFn)(const LLArgs);
template <int DT>
LLFn ll_pick_op(int op) {
  switch (op) {
    case BLINK_SUM: return ll_kernel<DT, BLINK_SUM>;
    case BLINK_PROD: return ll_kernel<DT, BLINK_PROD>;
    case BLINK_MIN: return ll_kernel<DT, BLINK_MIN>;
    case BLINK_MAX: return ll_kernel<DT, BLINK_MAX>;
    case BLINK_AVG: return ll_kernel<DT, BLINK_AVG>;
  }
  return nullptr;
}

cudaError_t launch_ll(const LLArgs& a, int grid, void* stream, bool cooperative, bool pdl) {
  LLFn fn = nullptr;
  if (a.coll == kBroadcast) {
    fn = ll_kernel<BLINK_FLOAT32, BLINK_SUM>;  // a byte copy
  } else {
    switch (a.dtype) {
      case BLINK_FLOAT32: fn = ll_pick_op<BLINK_FLOAT32>(a.op); break;
      case BLINK_BFLOAT16: fn = ll_pick_op<BLINK_BFLOAT16>(a.op); break;
      case BLINK_INT32: fn = ll_pick_op<BLINK_INT32>(a.op); break;
    }
  }
  if (!fn) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kLLThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  set_launch_attrs(cfg, attr, cooperative, pdl);
  return cudaLaunchKernelEx(&cfg, fn, a);
}

int exec_max_ctas_per_sm(int threads, bool vec, int dtype, int op, int coll, int smem_bytes) {
  ExecFn fn = pick(coll, dtype, op, vec);
  int n = 0;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, vec ? kMaxSmemBytes : 0);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, vec ? smem_bytes : 0) !=
      cudaSuccess)
    return 0;
  return n;
}

__global__ void store2_kernel(uint64_t* dst, uint64_t v0, uint64_t v1) {
  dst[1] = v1;
  __threadfence_system();
  dst[0] = v0;  // the tag last: a reader that sees it sees the value
}

cudaError_t launch_store2(uint64_t* dst, uint64_t v0, uint64_t v1, void* stream) {
  store2_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(dst, v0, v1);
  return cudaGetLastError();
}

// Load every kernel of the library on the current device now.  With lazy
// module loading (CUDA 12's default) the first launch of a kernel loads its
// module, which can wait for the device to go idle -- and a launch that
// spins on flags set by a LATER launch (per-rank launches, multi-process
// ranks sharing a GPU) would never let it.  Called once per device at comm
// creation.
cudaError_t preload_kernels() {
  cudaFuncAttributes fa;
  for (int coll = 0; coll <= kGather; ++coll)
    for (int dt = 0; dt < 3; ++dt)
      for (int op = 0; op <= BLINK_AVG; ++op)
        for (int vec = 0; vec < 2; ++vec) {
          ExecFn fn = pick(coll, dt, op, vec != 0);
          if (fn) {
            cudaError_t e = cudaFuncGetAttributes(&fa, fn);
            if (e != cudaSuccess) return e;
          }
        }
  for (int dt = 0; dt < 3; ++dt)
    for (int op = 0; op <= BLINK_AVG; ++op) {
      LLFn fn = dt == 0 ? ll_pick_op<BLINK_FLOAT32>(op)
                        : (dt == 1 ? ll_pick_op<BLINK_BFLOAT16>(op) : ll_pick_op<BLINK_INT32>(op));
      if (fn) {
        cudaError_t e = cudaFuncGetAttributes(&fa, fn);
        if (e != cudaSuccess) return e;
      }
    }
  cudaError_t e = cudaFuncGetAttributes(&fa, copy_kernel<true>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, copy_kernel<false>);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, store2_kernel);
  if (e == cudaSuccess) e = preload_nvls_kernels();
  return e;
}

cudaError_t launch_copy(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0 || dst == src) return cudaSuccess;
  bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t work = int64_t(bytes >> 4) / 512 + 1;
  int grid = int(work < int64_t(sms) * 4 ? work : int64_t(sms) * 4);
  if (vec)
    copy_kernel<true><<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<char*>(dst), static_cast<const char*>(src), int64_t(bytes));
  else
    copy_kernel<false><<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<char*>(dst), static_cast<const char*>(src), int64_t(bytes));
  return cudaGetLastError();
}

}  // namespace blink
