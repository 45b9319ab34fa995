// kernels.cu -- sm_100a kernels of the WSP hot path (libhetpipe).
//
// One fused, element-wise, HBM-streaming kernel per controller tick
// (tick_desc.h). No tensor cores: the path is a streaming reduction with < 0.2
// flop/byte; the design levers are 128-bit accesses, all loads
// of a chunk issued before any arithmetic (memory-level parallelism), streaming
// cache hints, a persistent grid sized from the occupancy calculator x 148 SMs,
// and fusing every op of a tick so each buffer crosses HBM at most once per tick.
//
// Rounding: every float op is an explicit __fmul_rn / __fadd_rn (no FMA
// contraction), which is the order and precision the paper's updates state
// (P:839 w_local + u_p, P:929 w_global + u~) under reading Z10.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>

#include "tick_desc.h"

namespace hp {
namespace {

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11): 10 rounds of two 32x32->64 multiplies
// and a Feistel-like mix, key bumped by the Weyl constants between rounds.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                               uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// FLOAT: (x>>8)*2^-24 - 0.5 ; DYADIC: (x>>28) - 8. Both exact in fp32.
template <int GM>
__device__ __forceinline__ float grad_of(uint32_t x) {
  if (GM == 1) return (float)((int)(x >> 28) - 8);
  return __fsub_rn(__fmul_rn((float)(x >> 8), 0x1p-24f), 0.5f);
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4scale(float s, float4 a) {
  return make_float4(__fmul_rn(s, a.x), __fmul_rn(s, a.y), __fmul_rn(s, a.z),
                     __fmul_rn(s, a.w));
}

// Chunk access: CNT == 4 is a full aligned float4; CNT < 4 the ragged tail
// (element-wise, zero-filled), only ever executed by one thread.
// HP_LD_VARIANT (compile time, tuning experiments): 0 = ld.global.cs (default),
// 1 = ld.global.cs.L2::256B, 2 = ld.global.L1::no_allocate.L2::256B, 3 = ld.global
#ifndef HP_LD_VARIANT
#define HP_LD_VARIANT 0
#endif
__device__ __forceinline__ float4 ldv4(const float4* p) {
#if HP_LD_VARIANT == 0
  return __ldcs(p);
#else
  float4 r;
#if HP_LD_VARIANT == 1
  asm volatile("ld.global.cs.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
#elif HP_LD_VARIANT == 2
  asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
#else
  asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
#endif
  return r;
#endif
}

template <int CNT>
__device__ __forceinline__ float4 ld4(const float* base, int64_t q) {
  if (CNT == 4) return ldv4(reinterpret_cast<const float4*>(base) + q);
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* p = base + 4 * q;
  r.x = p[0];
  if (CNT > 1) r.y = p[1];
  if (CNT > 2) r.z = p[2];
  return r;
}
template <int CNT>
__device__ __forceinline__ void st4(float* base, int64_t q, float4 v) {
  if (CNT == 4) {
    __stcs(reinterpret_cast<float4*>(base) + q, v);
    return;
  }
  float* p = base + 4 * q;
  p[0] = v.x;
  if (CNT > 1) p[1] = v.y;
  if (CNT > 2) p[2] = v.z;
}

// u = fl(-eta * g) for the 4 params of global block blk; -eta = the op's
// neg_lr (constant lr, or Theorem 1's eta_t = sigma / sqrt(t), host-computed).
template <int GM>
__device__ __forceinline__ float4 synth_u(const TickDesc& d, uint32_t v, uint32_t p,
                                          uint64_t blk, float nl) {
  const uint4 x = philox4x32_10((uint32_t)blk, v, p, 0u, d.key0, d.key1);
  return make_float4(__fmul_rn(nl, grad_of<GM>(x.x)), __fmul_rn(nl, grad_of<GM>(x.y)),
                     __fmul_rn(nl, grad_of<GM>(x.z)), __fmul_rn(nl, grad_of<GM>(x.w)));
}

// CONVEX (GM == 3): u = fl(-lr * fl(fl(a * fl(w - b)) + fl(sigma * xi))) with
// w = w_p (the weights minibatch p read at START), b = Philox stream 2
// (2*((x>>8)*2^-24) - 1), xi = the FLOAT draw of stream 0.
__device__ __forceinline__ float convex_u1(const TickDesc& d, float w, uint32_t xb, uint32_t xx,
                                           float nl) {
  const float b = __fsub_rn(__fmul_rn(2.0f, __fmul_rn((float)(xb >> 8), 0x1p-24f)), 1.0f);
  const float xi = __fsub_rn(__fmul_rn((float)(xx >> 8), 0x1p-24f), 0.5f);
  const float g = __fadd_rn(__fmul_rn(d.conv_a, __fsub_rn(w, b)), __fmul_rn(d.conv_sigma, xi));
  return __fmul_rn(nl, g);
}
__device__ __forceinline__ float4 convex_u(const TickDesc& d, uint32_t v, uint32_t p, uint64_t blk,
                                           float4 w, float nl) {
  const uint4 xb = philox4x32_10((uint32_t)blk, 0u, 0u, 2u, d.key0, d.key1);
  const uint4 xx = philox4x32_10((uint32_t)blk, v, p, 0u, d.key0, d.key1);
  return make_float4(convex_u1(d, w.x, xb.x, xx.x, nl), convex_u1(d, w.y, xb.y, xx.y, nl),
                     convex_u1(d, w.z, xb.z, xx.z, nl), convex_u1(d, w.w, xb.w, xx.w, nl));
}

// Source of chunk q among segments [b, e): first with 4q < end (ends are
// multiples of 32 params, so a chunk never straddles two segments).
__device__ __forceinline__ const float* seg_ptr(const TickDesc& d, int b, int e, int64_t q) {
  int s = b;
  while (s + 1 < e && 4 * q >= d.s[s].end) ++s;
  return d.s[s].ptr;
}

template <bool MOM>
__device__ __forceinline__ void apply(float4& wg, float4& m, float4 ut, float mu) {
  if (MOM) {
    m = f4add(f4scale(mu, m), ut);   // m = mu*m + u~   (Z11)
    wg = f4add(wg, m);               // w_global += m
  } else {
    wg = f4add(wg, ut);              // w_global += u~
  }
}

// Phase B of one complete: its loads (acc, inline-fold w_local, EXTERNAL
// gradient / CONVEX stash) ...
template <int GM, int U, int CNT>
__device__ __forceinline__ void complete_load(const DComplete& c, int64_t q0, int64_t qs,
                                              float4* ain, float4* win, float4* gin) {
  const uint32_t fl = c.flags;
#pragma unroll
  for (int x = 0; x < U; ++x) {
    const int64_t q = q0 + x * qs;
    if (fl & kLoadAcc) ain[x] = ld4<CNT>(c.acc, q);
    if (fl & kFoldInline) win[x] = ld4<CNT>(c.wl, q);
    if (GM == 2) gin[x] = ld4<CNT>(c.grad, q);
    if (GM == 3) gin[x] = ld4<CNT>(c.stash, q);             // w_p
  }
}
// ... and the rest: u, the wave aggregate, apply-now, inline fold.
template <int GM, bool MOM, int U, int CNT, bool LEAN = false>
__device__ __forceinline__ void complete_finish(const TickDesc& d, const DComplete& c, int64_t q0,
                                                int64_t qs, const float4* ain, const float4* win,
                                                const float4* gin, float4* wg, float4* mm) {
  const uint32_t fl = c.flags;
#pragma unroll
  for (int x = 0; x < U; ++x) {
    const int64_t q = q0 + x * qs;
    const uint64_t blk = (uint64_t)(d.blk_base + q);
    const float4 u = (GM == 2) ? f4scale(c.neg_lr, gin[x])
                     : (GM == 3) ? convex_u(d, c.v, c.p, blk, gin[x], c.neg_lr)
                                 : synth_u<GM>(d, c.v, c.p, blk, c.neg_lr);
    if (fl & kSnapAcc) st4<CNT>(c.snap, q, ain[x]);          // F > 1: acc at the gate
    const float4 a = (fl & kFirst) ? u : f4add(ain[x], u);   // wave aggregate
    if (fl & kStoreAcc) st4<CNT>(c.acc, q, a);
    if (!LEAN && (fl & kApplyNow)) apply<MOM>(wg[x], mm[x], a, d.mu);
    if (fl & kFoldInline) {
      const float4 w = f4add(win[x], u);
      st4<CNT>(c.wl, q, w);
      if (GM == 3 && (fl & kStashAfter)) st4<CNT>(c.stash, q, w);   // START(p+Nm)
    }
  }
}

// U chunks (4 params each), chunk x at q0 + x*qs, through phases A-D of
// tick_desc.h. Inside each op the loads of all U chunks are issued together,
// so a thread keeps U (or 2U-3U) 16-byte requests in flight per op while its
// register footprint stays independent of the number of ops in the tick.
template <int GM, bool MOM, int U, int CNT, bool LEAN = false>
__device__ __forceinline__ void tick_chunks(const TickDesc& d, int64_t q0, int64_t qs) {
  if constexpr (LEAN) {
    // completes only (no applies, w_global, groups or pull stores: Engine
    // picks this instance only for such launches): phase B alone, so the
    // w_global / momentum registers are never live -- fewer registers, more
    // CTAs per SM, more loads in flight for the 1-3 stream launches
    for (int j = 0; j < d.nc; ++j) {
      float4 ain[U], win[U], gin[U];
      complete_load<GM, U, CNT>(d.c[j], q0, qs, ain, win, gin);
      complete_finish<GM, false, U, CNT, true>(d, d.c[j], q0, qs, ain, win, gin, nullptr, nullptr);
    }
    return;
  }
  float4 wg[U], mm[U];
#pragma unroll
  for (int x = 0; x < U; ++x) {
    wg[x] = make_float4(0.f, 0.f, 0.f, 0.f);
    mm[x] = wg[x];
  }
  if (d.wg_load) {
#pragma unroll
    for (int x = 0; x < U; ++x) {
      const int64_t q = q0 + x * qs;
      wg[x] = ld4<CNT>(d.wgs_end > d.wgs_begin ? seg_ptr(d, d.wgs_begin, d.wgs_end, q) : d.wg, q);
    }
  }
  if (MOM && d.wg_store) {
#pragma unroll
    for (int x = 0; x < U; ++x) mm[x] = ld4<CNT>(d.m, q0 + x * qs);
  }
  // ---- A. memory-sourced applies, commit order ------------------------------
  int k0 = 0;
  if (U <= 2) {
    // two sources per step: twice the loads in flight per thread (the U = 2
    // launches carry the pulls and most applies); per element the applies
    // still run in commit order
    for (; k0 + 2 < d.na; k0 += 3) {
      float4 s0[U], s1[U], s2[U];
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int64_t q = q0 + x * qs;
        s0[x] = ld4<CNT>(seg_ptr(d, d.a[k0].seg_begin, d.a[k0].seg_end, q), q);
        s1[x] = ld4<CNT>(seg_ptr(d, d.a[k0 + 1].seg_begin, d.a[k0 + 1].seg_end, q), q);
        s2[x] = ld4<CNT>(seg_ptr(d, d.a[k0 + 2].seg_begin, d.a[k0 + 2].seg_end, q), q);
      }
#pragma unroll
      for (int x = 0; x < U; ++x) {
        apply<MOM>(wg[x], mm[x], s0[x], d.mu);
        apply<MOM>(wg[x], mm[x], s1[x], d.mu);
        apply<MOM>(wg[x], mm[x], s2[x], d.mu);
      }
    }
    for (; k0 + 1 < d.na; k0 += 2) {
      float4 s0[U], s1[U];
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int64_t q = q0 + x * qs;
        s0[x] = ld4<CNT>(seg_ptr(d, d.a[k0].seg_begin, d.a[k0].seg_end, q), q);
        s1[x] = ld4<CNT>(seg_ptr(d, d.a[k0 + 1].seg_begin, d.a[k0 + 1].seg_end, q), q);
      }
#pragma unroll
      for (int x = 0; x < U; ++x) {
        apply<MOM>(wg[x], mm[x], s0[x], d.mu);
        apply<MOM>(wg[x], mm[x], s1[x], d.mu);
      }
    }
  }
  for (int k = k0; k < d.na; ++k) {
    float4 s[U];
#pragma unroll
    for (int x = 0; x < U; ++x) s[x] = ld4<CNT>(seg_ptr(d, d.a[k].seg_begin, d.a[k].seg_end, q0 + x * qs), q0 + x * qs);
#pragma unroll
    for (int x = 0; x < U; ++x) apply<MOM>(wg[x], mm[x], s[x], d.mu);
  }
  // ---- B. completes --------------------------------------------------------
  // (pairing two completes' loads as in phase A needs ~45 more registers at
  // U = 2: it spills under the 4-CTA cap, so the completes stay sequential;
  // round 2 re-checked: 113 registers uncapped, 144 spilled bytes under the
  // 64-register cap; loading only the next complete's acc slot ahead spills
  // 48 bytes and ran 10% slower on C2's round-end launch, 6043 -> 5467 GB/s).
  // At U = 1 (the multi-tick kernel's chunks, the tails) registers are cheap:
  // two completes are loaded and drawn together, so their Philox chains
  // interleave -- the latency-bound C1 tick is two such chains long.
  int j0 = 0;
  if constexpr (U == 1) {
    for (; j0 + 1 < d.nc; j0 += 2) {
      float4 ain0[1], win0[1], gin0[1], ain1[1], win1[1], gin1[1];
      complete_load<GM, 1, CNT>(d.c[j0], q0, qs, ain0, win0, gin0);
      complete_load<GM, 1, CNT>(d.c[j0 + 1], q0, qs, ain1, win1, gin1);
      complete_finish<GM, MOM, 1, CNT>(d, d.c[j0], q0, qs, ain0, win0, gin0, wg, mm);
      complete_finish<GM, MOM, 1, CNT>(d, d.c[j0 + 1], q0, qs, ain1, win1, gin1, wg, mm);
    }
  }
  for (int j = j0; j < d.nc; ++j) {
    float4 ain[U], win[U], gin[U];
    complete_load<GM, U, CNT>(d.c[j], q0, qs, ain, win, gin);
    complete_finish<GM, MOM, U, CNT>(d, d.c[j], q0, qs, ain, win, gin, wg, mm);
  }
  // ---- C. store w_global / m ------------------------------------------------
  if (d.wg_store) {
#pragma unroll
    for (int x = 0; x < U; ++x) {
      st4<CNT>(d.wg, q0 + x * qs, wg[x]);
      if (MOM) st4<CNT>(d.m, q0 + x * qs, mm[x]);
    }
    // owner-side pull: the final w_global into every pulled w_local slice
    // (NVLink stores to the GPU that holds it; ranges are multiples of 32)
    for (int k = 0; k < d.np; ++k) {
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int64_t q = q0 + x * qs;
        if (4 * q >= d.pd[k].lo && 4 * q < d.pd[k].hi) st4<CNT>(d.pd[k].ptr, q, wg[x]);
      }
    }
  }
  // ---- D. w_local groups: pull base then due folds ---------
  for (int gi = 0; gi < d.ng; ++gi) {
    const DGroup& g = d.g[gi];
    float4 w[U];
#pragma unroll
    for (int x = 0; x < U; ++x) {
      const int64_t q = q0 + x * qs;
      if (g.pull == 0) w[x] = ld4<CNT>(g.wl, q);
      else if (g.pull == 2) w[x] = ld4<CNT>(seg_ptr(d, g.seg_begin, g.seg_end, q), q);
      else w[x] = wg[x];
      if (g.pull && g.partial) w[x] = f4add(w[x], ld4<CNT>(g.partial, q));
    }
    for (int fi = g.f_begin; fi < g.f_end; ++fi) {
      const DFold& f = d.f[fi];
      if (GM == 3 && f.op == 1) {                              // STASH: a START reads w
#pragma unroll
        for (int x = 0; x < U; ++x) st4<CNT>(f.stash, q0 + x * qs, w[x]);
        continue;
      }
      float4 sw[U];
      if (GM == 3) {
#pragma unroll
        for (int x = 0; x < U; ++x) sw[x] = ld4<CNT>(f.stash, q0 + x * qs);
      }
#pragma unroll
      for (int x = 0; x < U; ++x) {
        const int64_t q = q0 + x * qs;
        const uint64_t blk = (uint64_t)(d.blk_base + q);
        const float4 uf = (GM == 2) ? f4scale(f.neg_lr, ld4<CNT>(f.grad, q))
                          : (GM == 3) ? convex_u(d, f.v, f.p, blk, sw[x], f.neg_lr)
                                      : synth_u<GM>(d, f.v, f.p, blk, f.neg_lr);
        w[x] = f4add(w[x], uf);
      }
    }
#pragma unroll
    for (int x = 0; x < U; ++x) st4<CNT>(g.wl, q0 + x * qs, w[x]);
  }
}

// L2 prefetch (TickDesc::pf) of this CTA's tile of a later round: every buffer
// the round loads, one 4 KB contiguous bulk prefetch per (buffer, chunk x),
// spread over the CTA's threads. It costs no registers, so the bytes in flight
// per SM are no longer capped by the U loads each thread holds (launches with
// one or two load streams are latency-bound otherwise). Multi-segment sources
// are skipped (a hint only).
__device__ __forceinline__ void bulk_prefetch(const float* p) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(4096u) : "memory");
}
// NSEG 4 KB segments per buffer at chunks qb + x*S; (slot mod NL) == me issues.
template <int GM, bool MOM, int NSEG, int NL>
__device__ __forceinline__ void prefetch_round(const TickDesc& d, int64_t qb, int64_t S, int me) {
  int slot = 0;
  auto pf = [&](const float* base) {
#pragma unroll
    for (int x = 0; x < NSEG; ++x, ++slot)
      if ((slot % NL) == me) bulk_prefetch(base + 4 * (qb + x * S));
  };
  if (d.wg_load && d.wgs_end <= d.wgs_begin) pf(d.wg);
  if (MOM && d.wg_store) pf(d.m);
  for (int k = 0; k < d.na; ++k)
    if (d.a[k].seg_end - d.a[k].seg_begin == 1) pf(d.s[d.a[k].seg_begin].ptr);
  for (int j = 0; j < d.nc; ++j) {
    const DComplete& c = d.c[j];
    if (c.flags & kLoadAcc) pf(c.acc);
    if (c.flags & kFoldInline) pf(c.wl);
    if (GM == 2) pf(c.grad);
    if (GM == 3) pf(c.stash);
  }
  for (int gi = 0; gi < d.ng; ++gi) {
    const DGroup& g = d.g[gi];
    if (g.pull == 0) pf(g.wl);
    else if (g.pull == 2 && g.seg_end - g.seg_begin == 1) pf(d.s[g.seg_begin].ptr);
    if (g.pull && g.partial) pf(g.partial);
    for (int fi = g.f_begin; fi < g.f_end; ++fi) {
      if (GM == 2) pf(d.f[fi].grad);
      if (GM == 3 && d.f[fi].op != 1) pf(d.f[fi].stash);
    }
  }
}

template <int GM, bool MOM, int U, bool PF, bool DYN, bool LEAN = false>
__device__ __forceinline__ void tick_body(const TickDesc& d) {
  // Programmatic dependent launch: this grid may start while the previous tick
  // kernel drains; it touches no global memory before the previous grid has
  // completed and flushed its writes.
  cudaGridDependencySynchronize();
  const int64_t nfull = d.n >> 2;
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t q = t0;
  if (DYN) {
    // Dynamic tiles: tile k = chunks [k*256U, (k+1)*256U) (thread t takes
    // k*256U + x*256 + t: 4 KB contiguous per buffer and x), claimed from the
    // launch stream's counter by one thread per CTA two tiles ahead, so every
    // SM keeps streaming until the work runs out instead of idling behind the
    // slowest CTA of a static partition. (Per-warp claims of 512-byte runs
    // measured 7% slower: the DRAM wants the longer runs.) The last CTA to
    // finish zeroes the counters for the next launch on the stream.
    // Claiming the first tile too measured faster than starting CTA b on
    // tile b (C2 -4%).
    __shared__ long long nxt[3];
    const int64_t T = nfull / (256 * U);
    if (threadIdx.x == 0) {
      nxt[0] = (long long)atomicAdd(d.ctr, 1ull);
      nxt[1] = (long long)atomicAdd(d.ctr, 1ull);
    }
    __syncthreads();
    for (int j = 0;; j = j == 2 ? 0 : j + 1) {
      const int64_t k = nxt[j];
      if (k >= T) break;
      const int j1 = j == 2 ? 0 : j + 1, j2 = j1 == 2 ? 0 : j1 + 1;
      if (PF && nxt[j1] < T) prefetch_round<GM, MOM, U, 256>(d, nxt[j1] * 256 * U, 256, threadIdx.x);
      if (threadIdx.x == 0) nxt[j2] = (long long)atomicAdd(d.ctr, 1ull);
      tick_chunks<GM, MOM, U, 4, LEAN>(d, k * 256 * U + threadIdx.x, 256);
      __syncthreads();
    }
    for (q = T * 256 * U + t0; q < nfull; q += S) tick_chunks<GM, MOM, 1, 4, LEAN>(d, q, S);
  } else {
    const int64_t groups = nfull / (S * U);          // rounds where every thread has U chunks
    const int64_t cta0 = (int64_t)blockIdx.x * blockDim.x;   // this CTA's first chunk, round 0
    if (PF) {
      for (int64_t r = 1; r < d.pf && r < groups; ++r)
        prefetch_round<GM, MOM, U, 256>(d, cta0 + r * S * U, S, threadIdx.x);
      for (int64_t r = 0; r < groups; ++r, q += S * U) {
        if (r + d.pf < groups) prefetch_round<GM, MOM, U, 256>(d, cta0 + (r + d.pf) * S * U, S, threadIdx.x);
        tick_chunks<GM, MOM, U, 4, LEAN>(d, q, S);
      }
    } else {
      for (int64_t r = 0; r < groups; ++r, q += S * U) tick_chunks<GM, MOM, U, 4, LEAN>(d, q, S);
    }
    for (; q < nfull; q += S) tick_chunks<GM, MOM, 1, 4, LEAN>(d, q, S);
  }
  if (t0 == 0) {
    switch (d.n & 3) {
      case 1: tick_chunks<GM, MOM, 1, 1, LEAN>(d, nfull, 0); break;
      case 2: tick_chunks<GM, MOM, 1, 2, LEAN>(d, nfull, 0); break;
      case 3: tick_chunks<GM, MOM, 1, 3, LEAN>(d, nfull, 0); break;
      default: break;
    }
  }
  if (DYN && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(d.done, 1u) == gridDim.x - 1) {   // every CTA has made its last claim
      atomicExch(d.ctr, 0ull);
      atomicExch(d.done, 0u);
    }
  }
}

// The kernels: tick_body under the default register heuristics, and (tick_
// kernel_o4) capped for 4 resident CTAs per SM -- the dynamic-tile U = 2
// instances would otherwise drop to 3 (69 registers).
template <int GM, bool MOM, int U, bool PF, bool DYN>
__global__ void __launch_bounds__(256) tick_kernel(const __grid_constant__ TickDesc d) {
  tick_body<GM, MOM, U, PF, DYN>(d);
}
// (with momentum the U = 2 body spills 16 bytes under the 4-CTA cap; capping
// it for 3 CTAs/SM instead measured 3% slower on C5's momentum round-end
// launch, 4536 vs 4659 GB/s, profiles/r02/c5_1gpu_mom_cap.txt -- kept at 4)
#ifndef HP_MOM_O4_CTAS
#define HP_MOM_O4_CTAS 4
#endif
template <int GM, bool MOM, int U, bool PF, bool DYN>
__global__ void __launch_bounds__(256, (MOM ? HP_MOM_O4_CTAS : 4))
    tick_kernel_o4(const __grid_constant__ TickDesc d) {
  tick_body<GM, MOM, U, PF, DYN>(d);
}
// Completes-only launches (TickDesc::lean): phase B alone, capped for 4
// resident CTAs per SM (the general U = 4 instances hold 124 registers, 2 CTAs);
// 3 for the EXTERNAL / CONVEX gradients, which load one more stream per
// complete and would spill under 64 registers.
template <int GM, bool PF, bool DYN>
__global__ void __launch_bounds__(256, (GM >= 2 ? 3 : 4))
    tick_kernel_lean(const __grid_constant__ TickDesc d) {
  tick_body<GM, false, 4, PF, DYN, true>(d);
}

// Multi-tick kernel for launch-bound (small) models (hp_schedule_capture on a
// single-rank context, C1): `count` consecutive tick descriptors from device
// memory, run in order by ONE launch. Every op is element-wise in the param
// index (tick_desc.h), and each chunk of 4 params is owned by the same thread
// for all ticks (static stride, U = 1), so a thread's later tick sees its own
// earlier writes in program order -- no grid-wide synchronisation is needed;
// every tick still loads and stores exactly what its descriptor says. The
// descriptor of tick k is staged in shared memory (one coalesced 16-byte load
// per thread, issued during tick k-1), which replaces the chain of
// constant-cache misses a tiny one-tick launch spends its time in, and the code
// stays hot in the SMs' instruction caches across ticks (ncu on the one-tick
// C1 launches: stalls on instruction fetch dominate, 2.3 us active in 5.7 us).
template <int GM, bool MOM>
__global__ void __launch_bounds__(256) multi_tick_kernel(const TickDescPad* __restrict__ descs,
                                                         int count) {
  constexpr int kWords = (int)(sizeof(TickDescPad) / 16);
  static_assert(kWords <= 256, "one 16-byte word of the descriptor per thread");
  __shared__ __align__(16) uint4 sbuf[kWords];
  const TickDesc& sd = *reinterpret_cast<const TickDesc*>(sbuf);
  cudaGridDependencySynchronize();
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int w = threadIdx.x;
  uint4 nxt = make_uint4(0u, 0u, 0u, 0u);
  if (w < kWords && count > 0) nxt = __ldg(reinterpret_cast<const uint4*>(descs) + w);
  for (int k = 0; k < count; ++k) {
    if (w < kWords) sbuf[w] = nxt;
    __syncthreads();
    if (w < kWords && k + 1 < count)   // prefetch the next tick's descriptor
      nxt = __ldg(reinterpret_cast<const uint4*>(descs + k + 1) + w);
    const int64_t nfull = sd.n >> 2;
    for (int64_t q = t0; q < nfull; q += S) tick_chunks<GM, MOM, 1, 4>(sd, q, S);
    if (t0 == 0) {
      switch (sd.n & 3) {
        case 1: tick_chunks<GM, MOM, 1, 1>(sd, nfull, 0); break;
        case 2: tick_chunks<GM, MOM, 1, 2>(sd, nfull, 0); break;
        case 3: tick_chunks<GM, MOM, 1, 3>(sd, nfull, 0); break;
        default: break;
      }
    }
    __syncthreads();                   // every thread done with sbuf
  }
}

// ---------------------------------------------------------------------------
// NVLS lockstep exchange (NvlsDesc): the NVSwitch sums the N pushed u~ of this
// rank's shard range (multimem.ld_reduce, fp32 add in the switch), the owner
// adds the sum to w_global (one rounding: reading Z15) and multicasts the
// result into every GPU's w_local (multimem.st = the pull). One kernel
// replaces reduce-scatter + apply + all-gather.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 mc_ld_reduce4(const float* mc) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(mc)
               : "memory");
  return r;
}
__device__ __forceinline__ float mc_ld_reduce1(const float* mc) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(mc) : "memory");
  return r;
}
__device__ __forceinline__ void mc_st4(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               ::"l"(mc), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_st1(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}

// U chunks at q + x*stride: sum the shard's pushes in the switch, apply, and
// multicast the new w_global into every w_local.
template <int U>
__device__ __forceinline__ void nvls_chunks(const NvlsDesc& d, int64_t q, int64_t stride) {
  float4* wg4 = reinterpret_cast<float4*>(d.wg);
  float4 s[U], w[U];
#pragma unroll
  for (int x = 0; x < U; ++x) {
    s[x] = mc_ld_reduce4(d.mc_acc + 4 * (q + x * stride));
    w[x] = __ldcs(wg4 + q + x * stride);
  }
#pragma unroll
  for (int x = 0; x < U; ++x) {
    w[x] = f4add(w[x], s[x]);
    __stcs(wg4 + q + x * stride, w[x]);
    if (d.mc_wl) mc_st4(d.mc_wl + 4 * (q + x * stride), w[x]);
  }
}

template <int U, bool DYN>
__global__ void __launch_bounds__(256) nvls_kernel(const __grid_constant__ NvlsDesc d) {
  const int64_t nfull = d.n >> 2;
  const int64_t S = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t q = t0;
  if (DYN) {
    // dynamic tiles of 256U chunks claimed two ahead, as in tick_body
    __shared__ long long nxt[3];
    const int64_t T = nfull / (256 * U);
    if (threadIdx.x == 0) {
      nxt[0] = (long long)atomicAdd(d.ctr, 1ull);
      nxt[1] = (long long)atomicAdd(d.ctr, 1ull);
    }
    __syncthreads();
    for (int j = 0;; j = j == 2 ? 0 : j + 1) {
      const int64_t k = nxt[j];
      if (k >= T) break;
      if (threadIdx.x == 0) nxt[j == 0 ? 2 : j - 1] = (long long)atomicAdd(d.ctr, 1ull);
      nvls_chunks<U>(d, k * 256 * U + threadIdx.x, 256);
      __syncthreads();
    }
    q = T * 256 * U + t0;
  } else {
    for (; q + (U - 1) * S < nfull; q += U * S) nvls_chunks<U>(d, q, S);
  }
  for (; q < nfull; q += S) nvls_chunks<1>(d, q, 0);
  if (t0 == 0)
    for (int64_t i = nfull * 4; i < d.n; ++i) {
      const float w = __fadd_rn(d.wg[i], mc_ld_reduce1(d.mc_acc + i));
      d.wg[i] = w;
      if (d.mc_wl) mc_st1(d.mc_wl + i, w);
    }
  // the multicast stores must be visible system-wide before the barrier that
  // follows this kernel releases the other ranks to read their w_local
  __threadfence_system();
  if (DYN && threadIdx.x == 0 && atomicAdd(d.done, 1u) == gridDim.x - 1) {
    atomicExch(d.ctr, 0ull);
    atomicExch(d.done, 0u);
  }
}

// K7 barrier: lane q stores the epoch into rank q's flag slot of this rank
// (release, system scope: the writes of the kernels before it on this GPU are
// visible to any peer that sees the flag), then waits (acquire) until this
// rank's array holds the epoch from rank q. 10 s deadline (%globaltimer).
__global__ void flag_barrier_kernel(const __grid_constant__ FlagBarrier fb) {
  const int q = threadIdx.x;
  if (q < fb.G) {
    __threadfence_system();
    unsigned long long* dst = fb.flags[q] + fb.me;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(fb.epoch) : "memory");
    const unsigned long long* src = fb.flags[fb.me] + q;
    unsigned long long t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(src) : "memory");
      if (v >= fb.epoch) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > fb.timeout_ns) {
        if (fb.err) atomicExch(fb.err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// Point-to-point flags (FlagOps): lane i < nsig publishes val into sig[i]
// (release, system scope, after a system fence), lane i < nwait waits for
// wait[i] >= val (acquire); 10 s deadline as the barrier.
__global__ void flag_ops_kernel(const __grid_constant__ FlagOps fo) {
  const int i = threadIdx.x;
  if (i < fo.nsig) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fo.sig[i]), "l"(fo.val) : "memory");
  }
  if (i < fo.nwait) {
    unsigned long long t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(fo.wait[i]) : "memory");
      if (v >= fo.val) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > fo.timeout_ns) {
        if (fo.err && atomicExch(fo.err, 1) == 0) {   // first timeout: what it waited for
          fo.err[1] = (int)fo.val;
          fo.err[2] = (int)v;
          fo.err[3] = i;
          fo.err[4] = fo.nsig;
          fo.err[5] = fo.nwait;
        }
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// w0 (Z8): zero or Philox stream 1, counter (i>>2, 0, 0, 1).
__global__ void init_kernel(float* out, int64_t n, int64_t param_begin, int w0_mode,
                            int grad_mode, uint32_t k0, uint32_t k1) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t gi = param_begin + i;
    float w = 0.f;
    if (w0_mode == 1) {
      const uint4 x4 = philox4x32_10((uint32_t)(gi >> 2), 0u, 0u, 1u, k0, k1);
      const uint32_t words[4] = {x4.x, x4.y, x4.z, x4.w};
      const uint32_t x = words[gi & 3];
      if (grad_mode == 1) w = __fsub_rn(__fmul_rn((float)(x >> 25), 0x1p-6f), 1.0f);
      else w = __fsub_rn(__fmul_rn(2.0f, __fmul_rn((float)(x >> 8), 0x1p-24f)), 1.0f);
    }
    out[i] = w;
  }
}

int g_u_override = -1;   // HP_TICK_U: tuning override of chunks per thread
int g_pdl = 1;           // HP_PDL=0 disables programmatic dependent launch
int g_grid = 0;          // HP_GRID=1: one round of U chunks per thread (non-persistent)
int g_apply_u = 0;       // HP_APPLY_U: chunks per thread of launches with >= 2 applies

template <int GM, bool MOM, int U, bool PF, bool DYN, bool LEAN = false>
int launch_u(const TickDesc& d, cudaStream_t s, int max_blocks) {
  void (*kern)(const TickDesc);
  if constexpr (LEAN) kern = tick_kernel_lean<GM, PF, DYN>;
  else if constexpr (DYN && U == 2 && GM != 3) kern = tick_kernel_o4<GM, MOM, U, PF, DYN>;
  else kern = tick_kernel<GM, MOM, U, PF, DYN>;
  static int grid_max = 0;
  if (grid_max == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
    grid_max = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t chunks = (d.n + 3) >> 2;
  // max_blocks < 0: this launch non-persistent (one round of U chunks per
  // thread), so a higher-priority stream's kernel gets SMs as its CTAs retire
  const bool np = g_grid == 1 || max_blocks < 0;
  int64_t blocks = np ? (chunks + 256 * U - 1) / (256 * U) : (chunks + 255) / 256;
  if (!np && blocks > grid_max) blocks = grid_max;
  if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
  if (blocks > 0x7fffffff) blocks = 0x7fffffff;
  if (blocks < 1) blocks = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, kern, d);
}

template <int GM, bool MOM>
int launch_gm(const TickDesc& d, cudaStream_t s, int mb) {
  // Measured on B200 (profiles/): complete-only launches run best with 4 chunks
  // per thread; launches with pull groups (more ops per chunk, more Philox
  // folds) with 2, which keeps 3 CTAs/SM resident.
  int u = d.ng > 0 ? 2 : 4;
  // launches with >= 2 memory applies (the distributed owners' exchange: remote
  // u~ loads) at U = 2 take phase A's triple-source path: 3 sources x 2 chunks
  // in flight per thread at 4 CTAs/SM instead of 4 chunks of one source at 2
  // (HP_APPLY_U, tuning; 0 = as other launches)
  if (g_apply_u > 0 && d.na >= 2) u = g_apply_u;
  if (g_u_override > 0) u = g_u_override;
  // the L2 prefetch (d.pf > 0) is a separate instance, so the plain kernels keep
  // their code; the engine asks for it only on launches with few load streams
  // (complete-only, hence U = 4)
  const bool dyn = d.ctr != nullptr;
  if (u >= 4 && d.lean) {
    if (d.pf > 0) return dyn ? launch_u<GM, false, 4, true, true, true>(d, s, mb) : launch_u<GM, false, 4, true, false, true>(d, s, mb);
    return dyn ? launch_u<GM, false, 4, false, true, true>(d, s, mb) : launch_u<GM, false, 4, false, false, true>(d, s, mb);
  }
  if (u >= 4) {
    if (d.pf > 0) return dyn ? launch_u<GM, MOM, 4, true, true>(d, s, mb) : launch_u<GM, MOM, 4, true, false>(d, s, mb);
    return dyn ? launch_u<GM, MOM, 4, false, true>(d, s, mb) : launch_u<GM, MOM, 4, false, false>(d, s, mb);
  }
  return dyn ? launch_u<GM, MOM, 2, false, true>(d, s, mb) : launch_u<GM, MOM, 2, false, false>(d, s, mb);
}

}  // namespace

int launch_tick(const TickDesc& d, int grad_mode, bool momentum, void* stream, int mb) {
  cudaStream_t s = (cudaStream_t)stream;
  if (g_u_override == -1) {
    const char* e = getenv("HP_TICK_U");
    g_u_override = e ? atoi(e) : 0;
    const char* p = getenv("HP_PDL");
    g_pdl = p ? atoi(p) : 1;
    const char* g = getenv("HP_GRID");
    g_grid = g ? atoi(g) : 0;
    const char* au = getenv("HP_APPLY_U");
    g_apply_u = au ? atoi(au) : 0;
  }
  if (d.n <= 0) return 0;
  switch (grad_mode) {
    case 0: return momentum ? launch_gm<0, true>(d, s, mb) : launch_gm<0, false>(d, s, mb);
    case 1: return momentum ? launch_gm<1, true>(d, s, mb) : launch_gm<1, false>(d, s, mb);
    case 3: return momentum ? launch_gm<3, true>(d, s, mb) : launch_gm<3, false>(d, s, mb);
    default: return momentum ? launch_gm<2, true>(d, s, mb) : launch_gm<2, false>(d, s, mb);
  }
}

template <int U, bool DYN>
int launch_nvls_u(const NvlsDesc& d, cudaStream_t s, int max_blocks) {
  static int grid_max = 0;
  if (grid_max == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nvls_kernel<U, DYN>, 256, 0);
    grid_max = sms * (per_sm > 0 ? per_sm : 1);
  }
  int64_t blocks = ((d.n >> 2) + 255) / 256;
  if (blocks > grid_max) blocks = grid_max;
  if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  nvls_kernel<U, DYN><<<(unsigned)blocks, 256, 0, s>>>(d);
  return (int)cudaGetLastError();
}

int launch_multi_tick(const TickDescPad* descs, int count, int64_t n, int grad_mode, bool momentum,
                      void* stream) {
  if (count <= 0 || n <= 0) return 0;
  int64_t blocks = (((n + 3) >> 2) + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (grad_mode) {
    case 0: return (int)(momentum ? cudaLaunchKernelEx(&cfg, multi_tick_kernel<0, true>, descs, count)
                                  : cudaLaunchKernelEx(&cfg, multi_tick_kernel<0, false>, descs, count));
    case 1: return (int)(momentum ? cudaLaunchKernelEx(&cfg, multi_tick_kernel<1, true>, descs, count)
                                  : cudaLaunchKernelEx(&cfg, multi_tick_kernel<1, false>, descs, count));
    case 3: return (int)(momentum ? cudaLaunchKernelEx(&cfg, multi_tick_kernel<3, true>, descs, count)
                                  : cudaLaunchKernelEx(&cfg, multi_tick_kernel<3, false>, descs, count));
    default: return (int)cudaErrorInvalidValue;   // EXTERNAL gradients are never batched
  }
}

int launch_nvls(const NvlsDesc& d, void* stream, int max_blocks) {
  if (d.n <= 0) return 0;
  static int u = -1;   // HP_NVLS_U: multicast loads in flight per thread (2, 4, 8)
  if (u < 0) {
    const char* e = getenv("HP_NVLS_U");
    u = e ? atoi(e) : 4;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const bool dyn = d.ctr != nullptr;
  if (u >= 8) return dyn ? launch_nvls_u<8, true>(d, s, max_blocks) : launch_nvls_u<8, false>(d, s, max_blocks);
  if (u <= 2) return dyn ? launch_nvls_u<2, true>(d, s, max_blocks) : launch_nvls_u<2, false>(d, s, max_blocks);
  return dyn ? launch_nvls_u<4, true>(d, s, max_blocks) : launch_nvls_u<4, false>(d, s, max_blocks);
}

// HP_STRESS (race stress in place of compute-sanitizer):
// a one-warp kernel that idles for `ns` nanoseconds of %globaltimer, injected
// on a stream before a launch to perturb the relative timing of streams and
// ranks. It touches no memory.
__global__ void spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// Launch-floor probe (hp_launch_floor): an empty kernel launched like a tick
// kernel (one CTA of 256 threads, PDL attribute) -- the per-launch cost the
// latency-bound C1 ticks are compared with.
__global__ void __launch_bounds__(256) empty_kernel() { cudaGridDependencySynchronize(); }

int launch_empty(void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(256);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, empty_kernel);
}

int launch_spin(unsigned long long ns, void* stream) {
  spin_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ns);
  return (int)cudaGetLastError();
}

// Lazy module loading (the CUDA default) loads a kernel at its first launch,
// and a load may wait for the context to go idle. A flag barrier spinning on
// the device for a peer whose producer kernel is being loaded would then
// deadlock until the barrier's deadline (the CUDA guide's lazy-loading caveat
// for kernels that wait on each other) -- first seen with co-located ranks on
// one GPU. So every kernel instance the launchers can pick is loaded up front,
// once per device (cudaFuncGetAttributes forces the load).
template <int GM, bool MOM>
void preload_gm() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, tick_kernel<GM, MOM, 4, true, true>);
  cudaFuncGetAttributes(&a, tick_kernel<GM, MOM, 4, true, false>);
  cudaFuncGetAttributes(&a, tick_kernel<GM, MOM, 4, false, true>);
  cudaFuncGetAttributes(&a, tick_kernel<GM, MOM, 4, false, false>);
  if constexpr (GM != 3) cudaFuncGetAttributes(&a, tick_kernel_o4<GM, MOM, 2, false, true>);
  else cudaFuncGetAttributes(&a, tick_kernel<GM, MOM, 2, false, true>);
  cudaFuncGetAttributes(&a, tick_kernel<GM, MOM, 2, false, false>);
  if (!MOM) {
    cudaFuncGetAttributes(&a, tick_kernel_lean<GM, true, true>);
    cudaFuncGetAttributes(&a, tick_kernel_lean<GM, true, false>);
    cudaFuncGetAttributes(&a, tick_kernel_lean<GM, false, true>);
    cudaFuncGetAttributes(&a, tick_kernel_lean<GM, false, false>);
  }
}

int preload_kernels() {
  // once per device (module loading is per context; the caller has set the
  // device)
  static std::mutex mu;
  static unsigned long long done = 0;
  int dev = 0;
  if (int e = (int)cudaGetDevice(&dev)) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && (done >> dev) & 1ull) return 0;
  int err = 0;
  {
    cudaFuncAttributes a;
    preload_gm<0, false>();
    preload_gm<0, true>();
    preload_gm<1, false>();
    preload_gm<1, true>();
    preload_gm<2, false>();
    preload_gm<2, true>();
    preload_gm<3, false>();
    preload_gm<3, true>();
    for (auto k : {nvls_kernel<2, true>, nvls_kernel<2, false>, nvls_kernel<4, true>,
                   nvls_kernel<4, false>, nvls_kernel<8, true>, nvls_kernel<8, false>})
      cudaFuncGetAttributes(&a, k);
    cudaFuncGetAttributes(&a, flag_barrier_kernel);
    cudaFuncGetAttributes(&a, flag_ops_kernel);
    for (auto k : {multi_tick_kernel<0, false>, multi_tick_kernel<0, true>,
                   multi_tick_kernel<1, false>, multi_tick_kernel<1, true>,
                   multi_tick_kernel<3, false>, multi_tick_kernel<3, true>})
      cudaFuncGetAttributes(&a, k);
    cudaFuncGetAttributes(&a, spin_kernel);
    cudaFuncGetAttributes(&a, empty_kernel);
    cudaFuncGetAttributes(&a, init_kernel);
    err = (int)cudaGetLastError();
  }
  if (!err && dev < 64) done |= 1ull << dev;
  return err;
}

int launch_flag_barrier(const FlagBarrier& fb, void* stream) {
  flag_barrier_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(fb);
  return (int)cudaGetLastError();
}

int launch_flag_ops(const FlagOps& fo, void* stream) {
  flag_ops_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(fo);
  return (int)cudaGetLastError();
}

int launch_init(float* out, int64_t n, int64_t param_begin, int w0_mode, int grad_mode,
                uint32_t key0, uint32_t key1, void* stream) {
  if (n <= 0) return 0;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  init_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      out, n, param_begin, w0_mode, grad_mode, key0, key1);
  return (int)cudaGetLastError();
}

}  // namespace hp
