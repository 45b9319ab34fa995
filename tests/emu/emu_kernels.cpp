// TEST-ONLY host emulation of the tick descriptor semantics (tick_desc.h
// phases A-D) and of the w0 initialisation, scalar and sequential. Lets CPU
// tests check the engine's host logic against the oracle. Compiled with
// -ffp-contract=off so every float op rounds once, as __fadd_rn/__fmul_rn do.
#include <stdint.h>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2005_14038_b200/csrc/tick_desc.h"

namespace hp {
namespace {

void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
  }
}

float draw_u(const TickDesc& d, int gm, uint32_t v, uint32_t p, int64_t i, const float* grad,
             const float* stash, float nl) {
  if (gm == 2) return nl * grad[i];
  const int64_t gi = d.blk_base * 4 + i;
  uint32_t c[4] = {(uint32_t)(gi >> 2), v, p, 0u};
  philox(c, d.key0, d.key1);
  const uint32_t x = c[gi & 3];
  if (gm == 3) {                    // CONVEX: a (w_p - b) + sigma xi
    uint32_t cb[4] = {(uint32_t)(gi >> 2), 0u, 0u, 2u};
    philox(cb, d.key0, d.key1);
    const float b = 2.0f * ((float)(cb[gi & 3] >> 8) * 0x1p-24f) - 1.0f;
    const float xi = (float)(x >> 8) * 0x1p-24f - 0.5f;
    const float t1 = d.conv_a * (stash[i] - b);
    const float t2 = d.conv_sigma * xi;
    return nl * (t1 + t2);
  }
  const float g = gm == 1 ? (float)((int)(x >> 28) - 8) : (float)(x >> 8) * 0x1p-24f - 0.5f;
  return nl * g;
}

const float* seg(const TickDesc& d, int b, int e, int64_t i) {
  int s = b;
  while (s + 1 < e && i >= d.s[s].end) ++s;
  return d.s[s].ptr;
}

void app(const TickDesc& d, bool mom, float& wg, float& m, float ut) {
  if (mom) {
    m = d.mu * m + ut;
    wg = wg + m;
  } else {
    wg = wg + ut;
  }
}

}  // namespace

int launch_tick(const TickDesc& d, int gm, bool mom, void*, int) {
  for (int64_t i = 0; i < d.n; ++i) {
    float wg = !d.wg_load ? 0.f : d.wgs_end > d.wgs_begin ? seg(d, d.wgs_begin, d.wgs_end, i)[i] : d.wg[i];
    float m = (mom && d.wg_store) ? d.m[i] : 0.f;
    for (int k = 0; k < d.na; ++k) app(d, mom, wg, m, seg(d, d.a[k].seg_begin, d.a[k].seg_end, i)[i]);
    for (int j = 0; j < d.nc; ++j) {
      const DComplete& c = d.c[j];
      const float u = draw_u(d, gm, c.v, c.p, i, c.grad, c.stash, c.neg_lr);
      if (c.flags & kSnapAcc) c.snap[i] = c.acc[i];
      // (the acc is loaded only with kLoadAcc, as on the device: a fold-only
      // complete -- kFoldInline alone -- has no acc slot)
      const float a = (c.flags & kFirst) ? u : (c.flags & kLoadAcc) ? c.acc[i] + u : u;
      if (c.flags & kStoreAcc) c.acc[i] = a;
      if (c.flags & kApplyNow) app(d, mom, wg, m, a);
      if (c.flags & kFoldInline) {
        c.wl[i] = c.wl[i] + u;
        if (gm == 3 && (c.flags & kStashAfter)) c.stash[i] = c.wl[i];
      }
    }
    if (d.wg_store) {
      d.wg[i] = wg;
      if (mom) d.m[i] = m;
      for (int k = 0; k < d.np; ++k)
        if (i >= d.pd[k].lo && i < d.pd[k].hi) d.pd[k].ptr[i] = wg;
    }
    for (int g = 0; g < d.ng; ++g) {
      const DGroup& G = d.g[g];
      float w = G.pull == 0 ? G.wl[i] : G.pull == 2 ? seg(d, G.seg_begin, G.seg_end, i)[i] : wg;
      if (G.pull && G.partial) w = w + G.partial[i];
      for (int f = G.f_begin; f < G.f_end; ++f) {
        const DFold& F = d.f[f];
        if (gm == 3 && F.op == 1) F.stash[i] = w;            // STASH: a START reads w
        else w = w + draw_u(d, gm, F.v, F.p, i, F.grad, F.stash, F.neg_lr);
      }
      G.wl[i] = w;
    }
  }
  return 0;
}

// NVLS lockstep exchange through the unicast mappings: the switch's sum is
// emulated in rank order (the device order is the switch's, reading Z15).
int launch_nvls(const NvlsDesc& d, void*, int) {
  for (int64_t i = 0; i < d.n; ++i) {
    float s = d.src[0][i];
    for (int q = 1; q < d.G; ++q) s = s + d.src[q][i];
    const float w = d.wg[i] + s;
    d.wg[i] = w;
    if (d.mc_wl)
      for (int q = 0; q < d.G; ++q) d.dst[q][i] = w;
  }
  return 0;
}

int preload_kernels() { return 0; }
int launch_empty(void*) { return 0; }
int launch_multi_tick(const TickDescPad* descs, int count, int64_t, int grad_mode, bool momentum,
                      void* stream) {
  for (int k = 0; k < count; ++k)
    if (int e = launch_tick(descs[k].d, grad_mode, momentum, stream, 0)) return e;
  return 0;
}

// HP_STRESS spin: a no-op here (emulated kernels run at launch on the host)
int launch_spin(unsigned long long, void*) { return 0; }

// K7 flag barrier on host threads (ranks are threads of one process here)
int launch_flag_ops(const FlagOps& fo, void*) {
  for (int i = 0; i < fo.nsig; ++i) __atomic_store_n(fo.sig[i], fo.val, __ATOMIC_RELEASE);
  for (int i = 0; i < fo.nwait; ++i) {
    long spins = 0;
    while (__atomic_load_n(fo.wait[i], __ATOMIC_ACQUIRE) < fo.val) {
      if (++spins == 2000000000L && getenv("HP_EMU_DEBUG"))
        fprintf(stderr, "flag wait stuck: word %p val %llu have %llu\n", (void*)fo.wait[i],
                fo.val, (unsigned long long)__atomic_load_n(fo.wait[i], __ATOMIC_ACQUIRE));
    }
  }
  return 0;
}

int launch_flag_barrier(const FlagBarrier& fb, void*) {
  for (int q = 0; q < fb.G; ++q) __atomic_store_n(fb.flags[q] + fb.me, fb.epoch, __ATOMIC_RELEASE);
  for (int q = 0; q < fb.G; ++q)
    while (__atomic_load_n(fb.flags[fb.me] + q, __ATOMIC_ACQUIRE) < fb.epoch) {
    }
  return 0;
}

int launch_init(float* out, int64_t n, int64_t begin, int w0_mode, int gm, uint32_t k0,
                uint32_t k1, void*) {
  for (int64_t i = 0; i < n; ++i) {
    const int64_t gi = begin + i;
    float w = 0.f;
    if (w0_mode == 1) {
      uint32_t c[4] = {(uint32_t)(gi >> 2), 0u, 0u, 1u};
      philox(c, k0, k1);
      const uint32_t x = c[gi & 3];
      w = gm == 1 ? (float)(x >> 25) * 0x1p-6f - 1.0f : 2.0f * ((float)(x >> 8) * 0x1p-24f) - 1.0f;
    }
    out[i] = w;
  }
  return 0;
}

}  // namespace hp
