// What one tree hop costs, part by part, on one B200 (scripts/hop_trace.py
// measured ~3.5 us per hop for a 4 KB chunk: 1.1 us load-to-store, 1.4 us
// store completion, 0.8 us signal-to-load).  Each test runs N times in one
// thread (or warp) of one CTA on L2-resident data and reports the mean in ns
// (%globaltimer) and SM cycles (clock64).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hop_parts scripts/hop_parts_probe.cu
//   /tmp/hop_parts
//
//   tma_load      cp.async.bulk global->smem of B bytes, wait on its mbarrier
//   tma_store     cp.async.bulk smem->global of B bytes, commit, wait_group 0
//   tma_store_rd  the same, wait_group.read 0 (smem reusable, writes not done)
//   lsu_store     one warp stores B bytes (16 B per lane per step) + __syncwarp
//                 + fence.acq_rel.gpu by lane 0
//   fence_acqrel  fence.acq_rel.gpu alone
//   fence_proxy   fence.proxy.async alone
//   pingpong_*    two CTAs bounce a flag N times; one-way latency
//                 relaxed: st.relaxed.gpu + fence / ld.relaxed.gpu poll + fence
//                 relacq:  st.release.gpu / ld.acquire.gpu poll
//                 volatile: st.volatile / ld.volatile poll (+ __threadfence)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

constexpr int N = 200;

__global__ void parts(char* buf, int bytes, unsigned long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // warm the lines into L2
  for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16) *reinterpret_cast<uint4*>(buf + i) = make_uint4(i, 0, 0, 0);
  __syncthreads();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (threadIdx.x >= 32) return;
  uint64_t t0, t1;
  long long c0, c1;
  // tma_load
  if (lane == 0) {
    t0 = gtimer();
    c0 = clock64();
    for (int i = 0; i < N; ++i) {
      mbar_expect_tx(&bar, bytes);
      tma_load(sm, buf, bytes, &bar);
      mbar_wait(&bar, i & 1);
    }
    c1 = clock64();
    t1 = gtimer();
    out[0] = (t1 - t0);
    out[1] = (c1 - c0);
  }
  __syncwarp();
  // tma_store + wait_group 0
  if (lane == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    t0 = gtimer();
    c0 = clock64();
    for (int i = 0; i < N; ++i) {
      tma_store(buf + bytes, sm, bytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    c1 = clock64();
    t1 = gtimer();
    out[2] = (t1 - t0);
    out[3] = (c1 - c0);
    t0 = gtimer();
    c0 = clock64();
    for (int i = 0; i < N; ++i) {
      tma_store(buf + bytes, sm, bytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    c1 = clock64();
    t1 = gtimer();
    out[4] = (t1 - t0);
    out[5] = (c1 - c0);
  }
  __syncwarp();
  // lsu_store: whole warp
  {
    const uint4* s4 = reinterpret_cast<const uint4*>(sm);
    uint4* d4 = reinterpret_cast<uint4*>(buf + 2 * bytes);
    t0 = gtimer();
    c0 = clock64();
    for (int i = 0; i < N; ++i) {
      for (int k = lane; k < bytes / 16; k += 32) d4[k] = s4[k];
      __syncwarp();
      if (lane == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      __syncwarp();
    }
    c1 = clock64();
    t1 = gtimer();
    if (lane == 0) {
      out[6] = (t1 - t0);
      out[7] = (c1 - c0);
    }
  }
  if (lane == 0) {
    t0 = gtimer();
    c0 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    c1 = clock64();
    t1 = gtimer();
    out[8] = (t1 - t0);
    out[9] = (c1 - c0);
    t0 = gtimer();
    c0 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("fence.proxy.async;" ::: "memory");
    c1 = clock64();
    t1 = gtimer();
    out[10] = (t1 - t0);
    out[11] = (c1 - c0);
  }
}

template <int MODE>
__global__ void pingpong(uint64_t* flags, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  uint64_t* mine = flags + (blockIdx.x == 0 ? 0 : 32);
  uint64_t* theirs = flags + (blockIdx.x == 0 ? 32 : 0);
  const uint64_t t0 = gtimer();
  for (uint64_t i = 1; i <= N; ++i) {
    if (blockIdx.x == 1) {  // wait first
      for (;;) {
        uint64_t v;
        if (MODE == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        else if (MODE == 1) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        else v = *reinterpret_cast<volatile uint64_t*>(mine);
        if (v >= i) break;
      }
      if (MODE != 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    if (MODE == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(theirs), "l"(i) : "memory");
    } else if (MODE == 1) {
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(theirs), "l"(i) : "memory");
    } else {
      __threadfence();
      *reinterpret_cast<volatile uint64_t*>(theirs) = i;
    }
    if (blockIdx.x == 0) {
      for (;;) {
        uint64_t v;
        if (MODE == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        else if (MODE == 1) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        else v = *reinterpret_cast<volatile uint64_t*>(mine);
        if (v >= i) break;
      }
      if (MODE != 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  }
  if (blockIdx.x == 0) out[MODE] = gtimer() - t0;
}


// Two CTAs bounce a B-byte chunk with the executor's primitives: wait flag
// (relaxed poll + fence.acq_rel) -> fence.proxy.async -> TMA load of the
// chunk (written by the other CTA's bulk store) -> TMA store into the other
// CTA's buffer -> wait_group 0 -> fence.proxy.async -> fence.acq_rel ->
// relaxed flag store.  One-way time = one hop of a path.  VAR 1: the flag is
// st.release / ld.acquire; VAR 2: the load / store are done by the warp
// with LSU (ld.global.cg / st.global) instead of TMA.
template <int VAR>
__global__ void hop_pingpong(char* bufs, uint64_t* flags, int bytes, unsigned long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x;
  const int me = blockIdx.x, other = 1 - me;
  char* mybuf = bufs + size_t(me) * (1 << 20);
  char* obuf = bufs + size_t(other) * (1 << 20);
  uint64_t* myflag = flags + me * 32;
  uint64_t* oflag = flags + other * 32;
  if (lane == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t t0 = gtimer();
  for (uint64_t i = 1; i <= N; ++i) {
    if (!(me == 0 && i == 1)) {
      if (lane == 0) {
        for (;;) {
          uint64_t v;
          if (VAR == 1) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(myflag) : "memory");
          else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(myflag) : "memory");
          if (v >= i - (me == 0 ? 1 : 0)) break;
        }
        if (VAR != 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncwarp();
    }
    if (VAR == 2) {
      const uint4* s4 = reinterpret_cast<const uint4*>(mybuf);
      uint4* d4 = reinterpret_cast<uint4*>(obuf);
      for (int k = lane; k < bytes / 16; k += 32) d4[k] = __ldcg(s4 + k);
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(oflag), "l"(i) : "memory");
      }
      __syncwarp();
      continue;
    }
    if (lane == 0) {
      asm volatile("fence.proxy.async;" ::: "memory");
      mbar_expect_tx(&bar, bytes);
      tma_load(sm, mybuf, bytes, &bar);
      mbar_wait(&bar, (i - 1) & 1);
      tma_store(obuf, sm, bytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async;" ::: "memory");
      if (VAR == 1) {
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(oflag), "l"(i) : "memory");
      } else {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(oflag), "l"(i) : "memory");
      }
    }
    __syncwarp();
  }
  if (me == 0 && lane == 0) out[VAR] = gtimer() - t0;
}


// VAR 0: the hop split like the executor -- warp 0 lane 0 polls the flag and
// issues the TMA load; warp 1 lane 0 waits on the stage mbarrier (try_wait,
// or test_wait spin for VAR 1), bulk-stores, drains and signals.
template <int VAR>
__global__ void hop_split(char* bufs, uint64_t* flags, int bytes, unsigned long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t full;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int me = blockIdx.x, other = 1 - me;
  char* mybuf = bufs + size_t(me) * (1 << 20);
  char* obuf = bufs + size_t(other) * (1 << 20);
  uint64_t* myflag = flags + me * 32;
  uint64_t* oflag = flags + other * 32;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t t0 = gtimer();
  for (uint64_t i = 1; i <= N; ++i) {
    const uint64_t want = i - (me == 0 ? 1 : 0);
    if (warp == 0 && lane == 0) {
      if (!(me == 0 && i == 1)) {
        for (;;) {
          uint64_t v;
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(myflag) : "memory");
          if (v >= want) break;
        }
      }
      asm volatile("fence.proxy.async;" ::: "memory");
      mbar_expect_tx(&full, bytes);
      tma_load(sm, mybuf, bytes, &full);
    } else if (warp == 1 && lane == 0) {
      if (VAR == 0) {
        mbar_wait(&full, (i - 1) & 1);
      } else {
        for (;;) {
          uint32_t done;
          asm volatile(
              "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done)
              : "r"(smem_u32(&full)), "r"(uint32_t((i - 1) & 1))
              : "memory");
          if (done) break;
        }
      }
      tma_store(obuf, sm, bytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async;" ::: "memory");
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(oflag), "l"(i) : "memory");
    }
    __syncthreads();
  }
  if (me == 0 && threadIdx.x == 0) out[8 + VAR] = gtimer() - t0;
}


// A chain over G CTAs, each used ONCE (like the executor's per-call hops):
// CTA k waits for flag k, moves the B-byte chunk from buffer k to buffer k+1
// (TMA: one thread loads + stores; VAR 1: the warp with 16-byte LSU copies)
// and raises flag k+1.  Time per hop = (end - start) / (G - 1).
template <int VAR>
__global__ void hop_chain(char* bufs, uint64_t* flags, int bytes, unsigned long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t full;
  const int k = blockIdx.x, lane = threadIdx.x;
  char* src = bufs + size_t(k) * 65536;
  char* dst = bufs + size_t(k + 1) * 65536;
  if (lane == 0) {
    mbar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (k == 0 && lane == 0) out[12 + VAR] = gtimer();
  if (k > 0 && lane == 0) {
    for (;;) {
      uint64_t v;
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + 32 * k) : "memory");
      if (v) break;
    }
  }
  __syncwarp();
  if (VAR == 0) {
    if (lane == 0) {
      asm volatile("fence.proxy.async;" ::: "memory");
      mbar_expect_tx(&full, bytes);
      tma_load(sm, src, bytes, &full);
      mbar_wait(&full, 0);
      tma_store(dst, sm, bytes);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async;" ::: "memory");
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + 32 * (k + 1)), "l"(1ull) : "memory");
    }
  } else {
    for (int j = lane; j < bytes / 16; j += 32)
      reinterpret_cast<uint4*>(dst)[j] = __ldcg(reinterpret_cast<const uint4*>(src) + j);
    __syncwarp();
    if (lane == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + 32 * (k + 1)), "l"(1ull) : "memory");
  }
  if (k == gridDim.x - 1 && lane == 0) out[14 + VAR] = gtimer();
}


// Instruction fetch: one thread runs 4096 straight-line IADDs (64 KB of SASS)
// twice; pass 1 fetches the code cold from L2, pass 2 runs from the
// instruction caches.  Independent adds over 8 registers (no dependency
// stalls beyond issue).
#define MIX(r) "{ .reg .b32 t; mul.lo.u32 " r ", " r ", 0x9e3779b1; shr.b32 t, " r ", 13; xor.b32 " r ", " r ", t; }"
#define ADD8 asm volatile(MIX("%0") MIX("%1") MIX("%2") MIX("%3") MIX("%4") MIX("%5") MIX("%6") MIX("%7") : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3), "+r"(r4), "+r"(r5), "+r"(r6), "+r"(r7));
#define ADD64 ADD8 ADD8 ADD8 ADD8 ADD8 ADD8 ADD8 ADD8
#define ADD512 ADD64 ADD64 ADD64 ADD64 ADD64 ADD64 ADD64 ADD64
__global__ void icache_probe(unsigned long long* out) {
  if (threadIdx.x != 0) return;
  uint32_t r0 = clock(), r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  long long c[3];
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c[pass]) :: "memory");
    ADD512 ADD512 ADD512
  }
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c[2]) :: "memory");
  out[0] = c[1] - c[0];
  out[1] = c[2] - c[1];
  out[2] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}


// The same one-shot chain, every CTA's buffer in its own allocation (distinct
// 2 MB pages, like the executor's per-rank buffers and flag regions); VAR 1
// first touches its source and destination with a 16-byte TMA prefetch /
// generic load before waiting on its flag (translation warm-up).
template <int VAR>
__global__ void hop_chain_pages(char* const* bufs, uint64_t* const* flags, int bytes, unsigned long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t full;
  const int k = blockIdx.x, lane = threadIdx.x;
  char* src = bufs[k];
  char* dst = bufs[k + 1];
  if (lane == 0) {
    mbar_init(&full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (VAR == 1) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], 16;" ::"l"(src) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], 16;" ::"l"(dst) : "memory");
    }
  }
  __syncwarp();
  if (k == 0 && lane == 0) out[12 + VAR] = gtimer();
  if (k > 0 && lane == 0) {
    for (;;) {
      uint64_t v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags[k]) : "memory");
      if (v) break;
    }
    asm volatile("fence.acquire.gpu;" ::: "memory");
  }
  __syncwarp();
  if (lane == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(&full, bytes);
    tma_load(sm, src, bytes, &full);
    mbar_wait(&full, 0);
    tma_store(dst, sm, bytes);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags[k + 1]), "l"(1ull) : "memory");
  }
  if (k == gridDim.x - 1 && lane == 0) out[14 + VAR] = gtimer();
}


// The one-shot chain with the executor's CTA shape: 256 threads, 200 KB of
// dynamic shared memory, warp 0 = producer (lane 0 polls, fence, TMA load
// into stage 0 with an mbarrier, then posts an end-of-stream meta into stage
// 1), warp 1 lane 0 = store thread (waits stage 0, bulk-stores, waits the
// end-of-stream, drains, publishes); the other warps wait at __syncthreads.
struct PMeta { int c, tb; };
__global__ void __launch_bounds__(256, 1) hop_chain_exec(char* const* bufs, uint64_t* const* flags, int bytes,
                                                          unsigned long long* out, unsigned long long* cyc) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t full[2];
  __shared__ PMeta meta[2];
  const int k = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* src = bufs[k];
  char* dst = bufs[k + 1];
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (k == 0 && threadIdx.x == 0) out[12] = gtimer();
  if (warp == 0) {
    if (k > 0 && lane == 0) {
      for (;;) {
        uint64_t v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags[k]) : "memory");
        if (v) break;
      }
      asm volatile("fence.acquire.gpu;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0 && k == 3) cyc[1] = gtimer();
    if (lane == 0 && k == 4) cyc[8] = gtimer();
    if (lane == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (k == 3) cyc[2] = gtimer();
      meta[0].c = 0;
      meta[0].tb = bytes;
      mbar_expect_tx(&full[0], bytes);
      tma_load(ring, src, bytes, &full[0]);
      meta[1].c = -1;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[1])) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    mbar_wait(&full[0], 0);
    const uint64_t t_full = gtimer();
    tma_store(dst, ring, uint32_t(meta[0].tb));
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    const uint64_t t_store = gtimer();
    mbar_wait(&full[1], 0);
    const uint64_t t_eos = gtimer();
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    const uint64_t t_drained = gtimer();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const long long c0 = clock64();
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags[k + 1]), "l"(1ull) : "memory");
    const long long c1 = clock64();
    const uint64_t t_pub = gtimer();
    if (k == 3) {
      cyc[0] = c1 - c0;
      cyc[3] = t_full; cyc[4] = t_store; cyc[5] = t_eos; cyc[6] = t_drained; cyc[7] = t_pub;
    }
  }
  __syncthreads();
  if (k == gridDim.x - 1 && threadIdx.x == 0) out[14] = gtimer();
}

int main() {
  char* buf;
  unsigned long long *out, h[16];
  uint64_t* flags;
  cudaMalloc(&buf, 1 << 24);
  cudaMalloc(&out, 16 * sizeof(unsigned long long));
  cudaMalloc(&flags, 4096);
  cudaFuncSetAttribute(parts, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10);
  for (int bytes : {4096, 16384, 65536}) {
    parts<<<1, 256, 65536 + 1024>>>(buf, bytes, out);
    parts<<<1, 256, 65536 + 1024>>>(buf, bytes, out);
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"tma_load", "tma_store", "tma_store_rd", "lsu_store+fence", "fence_acqrel", "fence_proxy"};
    printf("B = %d\n", bytes);
    for (int k = 0; k < 6; ++k)
      printf("  %-16s %8.1f ns %8.1f cyc\n", names[k], double(h[2 * k]) / N, double(h[2 * k + 1]) / N);
  }
  const char* pn[] = {"relaxed+fence", "release/acquire", "volatile+threadfence"};
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(flags, 0, 4096);
    pingpong<0><<<2, 32>>>(flags, out);
    cudaMemset(flags, 0, 4096);
    pingpong<1><<<2, 32>>>(flags, out);
    cudaMemset(flags, 0, 4096);
    pingpong<2><<<2, 32>>>(flags, out);
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  }
  for (int k = 0; k < 3; ++k) printf("pingpong %-22s one-way %8.1f ns\n", pn[k], double(h[k]) / N / 2);
  char* hb;
  cudaMalloc(&hb, 2 << 20);
  cudaMemset(hb, 1, 2 << 20);
  const char* hn[] = {"tma relaxed+fence", "tma release/acquire", "lsu relaxed+fence"};
  cudaFuncSetAttribute(hop_pingpong<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(hop_pingpong<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(hop_pingpong<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaMemset(out, 0, 16 * sizeof(unsigned long long));
  for (int kind : {0, 1}) {  // 0: both CTAs on nearby SMs; 1: grid of 148, CTAs 0 and 147 bounce
    for (int bytes : {4096, 16384, 65536}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(flags, 0, 4096);
        hop_pingpong<0><<<2, 32, 65536>>>(hb, flags, bytes, out);
        cudaMemset(flags, 0, 4096);
        hop_pingpong<1><<<2, 32, 65536>>>(hb, flags, bytes, out);
        cudaMemset(flags, 0, 4096);
        hop_pingpong<2><<<2, 32, 65536>>>(hb, flags, bytes, out);
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      for (int k = 0; k < 3; ++k) printf("hop B=%6d %-22s one-way %8.1f ns\n", bytes, hn[k], double(h[k]) / N / 2);
      printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
    }
    break;
  }
  cudaFuncSetAttribute(hop_split<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(hop_split<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int bytes : {4096, 16384, 65536}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(flags, 0, 4096);
      hop_split<0><<<2, 256, 65536>>>(hb, flags, bytes, out);
      cudaMemset(flags, 0, 4096);
      hop_split<1><<<2, 256, 65536>>>(hb, flags, bytes, out);
    }
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("hop B=%6d split warps, try_wait      one-way %8.1f ns\n", bytes, double(h[8]) / N / 2);
    printf("hop B=%6d split warps, test_wait spin one-way %8.1f ns\n", bytes, double(h[9]) / N / 2);
  }
  {
    char* cb;
    uint64_t* cf;
    const int G = 100;
    cudaMalloc(&cb, size_t(G + 1) * 65536);
    cudaMalloc(&cf, size_t(G + 1) * 256);
    cudaMemset(cb, 3, size_t(G + 1) * 65536);
    cudaFuncSetAttribute(hop_chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(hop_chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int bytes : {4096, 16384, 65536}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(cf, 0, size_t(G + 1) * 256);
        hop_chain<0><<<G, 32, 65536>>>(cb, cf, bytes, out);
        cudaMemset(cf, 0, size_t(G + 1) * 256);
        hop_chain<1><<<G, 32, 65536>>>(cb, cf, bytes, out);
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      printf("chain of %d CTAs (each once) B=%6d: TMA %7.1f ns/hop, LSU warp %7.1f ns/hop\n", G, bytes,
             double(h[14] - h[12]) / (G - 1), double(h[15] - h[13]) / (G - 1));
    }
  }
  {
    const int G = 100;
    std::vector<char*> hb2(G + 1);
    std::vector<uint64_t*> hf(G + 1);
    for (int i = 0; i <= G; ++i) {
      cudaMalloc(&hb2[i], 4 << 20);
      cudaMalloc(&hf[i], 4 << 20);
      cudaMemset(hb2[i], 1, 65536);
    }
    char** db;
    uint64_t** df;
    cudaMalloc(&db, sizeof(char*) * (G + 1));
    cudaMalloc(&df, sizeof(uint64_t*) * (G + 1));
    cudaMemcpy(db, hb2.data(), sizeof(char*) * (G + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(df, hf.data(), sizeof(uint64_t*) * (G + 1), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(hop_chain_pages<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(hop_chain_pages<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int bytes : {4096, 65536}) {
      for (int rep = 0; rep < 3; ++rep) {
        for (int i = 0; i <= G; ++i) cudaMemset(hf[i], 0, 64);
        hop_chain_pages<0><<<G, 32, 65536>>>(db, df, bytes, out);
        for (int i = 0; i <= G; ++i) cudaMemset(hf[i], 0, 64);
        hop_chain_pages<1><<<G, 32, 65536>>>(db, df, bytes, out);
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      printf("chain, separate 4 MB allocations, B=%6d: TMA %7.1f ns/hop, with prefetch first %7.1f ns/hop\n", bytes,
             double(h[14] - h[12]) / (G - 1), double(h[15] - h[13]) / (G - 1));
    }
  }
  {
    const int G = 100;
    std::vector<char*> hb3(G + 1);
    std::vector<uint64_t*> hf3(G + 1);
    for (int i = 0; i <= G; ++i) {
      cudaMalloc(&hb3[i], 4 << 20);
      cudaMalloc(&hf3[i], 4 << 20);
      cudaMemset(hb3[i], 1, 65536);
    }
    char** db;
    uint64_t** df;
    unsigned long long* dc;
    cudaMalloc(&db, sizeof(char*) * (G + 1));
    cudaMalloc(&df, sizeof(uint64_t*) * (G + 1));
    cudaMalloc(&dc, 256);
    cudaMemcpy(db, hb3.data(), sizeof(char*) * (G + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(df, hf3.data(), sizeof(uint64_t*) * (G + 1), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(hop_chain_exec, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    for (int bytes : {4096, 65536}) {
      unsigned long long hc = 0;
      for (int rep = 0; rep < 3; ++rep) {
        for (int i = 0; i <= G; ++i) cudaMemset(hf3[i], 0, 64);
        hop_chain_exec<<<G, 256, 200 << 10>>>(db, df, bytes, out, dc);
      }
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
      printf("chain, executor CTA shape (256 thr, 200 KB smem, producer/store warps), B=%6d: %7.1f ns/hop, publish %llu cyc (%s)\n",
             bytes, double(h[14] - h[12]) / (G - 1), hc, cudaGetErrorString(cudaGetLastError()));
      unsigned long long hs[8 + 1];
      cudaMemcpy(hs, dc, sizeof(hs), cudaMemcpyDeviceToHost);
      const double b0 = double(hs[9]);
      printf("  CTA 3 (ns from acquire): issue %.0f full %.0f store %.0f eos %.0f drained %.0f published %.0f; CTA 4 acquired %.0f\n",
             double(hs[2]) - double(hs[1]), double(hs[3]) - double(hs[1]), double(hs[4]) - double(hs[1]),
             double(hs[5]) - double(hs[1]), double(hs[6]) - double(hs[1]), double(hs[7]) - double(hs[1]),
             double(hs[8]) - double(hs[1]));
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    icache_probe<<<1, 32>>>(out);
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("icache: 4608 ALU instructions (~74 KB SASS) pass 1 (cold) %lld cyc, pass 2 (warm) %lld cyc\n",
           (long long)h[0], (long long)h[1]);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
