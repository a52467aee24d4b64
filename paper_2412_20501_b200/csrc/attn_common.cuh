// Shared device pieces of the sm_100a attention kernels (attn_fwd_sm100.cu:
// the product kernel; attn_fwd_variants.cu: measured alternatives): tile
// configuration, the per-CTA kv-tile walk, the CTA -> (head, q tile) map,
// the softmax exp2 -> P emitter, and the host-side launch hooks.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>

#include "tr_internal.h"
#include "tr_ptx.cuh"

namespace tr {

template <int D>
struct AttnCfg {
  static constexpr int BM = 128;  // rows per half
  static constexpr int BN = 128;  // keys per kv tile
  static constexpr int NB = D / 64;               // 64-column TMA boxes per tile row
  static constexpr int BOX = 128 * 64 * 2;        // bytes per box (16 KB)
  static constexpr int TILE = NB * BOX;           // bytes per 128-row tile
#ifndef TR_NS128
#define TR_NS128 4
#endif
  static constexpr int NS = (D == 128) ? TR_NS128 : 6;   // kv ring stages (K and V alternate)
  static constexpr int THREADS = 384;
  static constexpr int SMEM_TILES = (2 + NS) * TILE;
  static constexpr int SMEM = SMEM_TILES + 1024 /*barriers*/ + 1024 /*alignment slack*/;
  static constexpr uint32_t IDESC_QK = idesc_bf16(128, BN, false);
  static constexpr uint32_t IDESC_PV = idesc_bf16(128, D, true);
  static constexpr float RESCALE_LOG2 = 8.0f;
#ifndef TR_POLY_MOD
#define TR_POLY_MOD 6
#endif
  static constexpr int POLY_MOD = TR_POLY_MOD;   // 1 of every POLY_MOD exp2 pairs on the FMA pipe
#ifndef TR_P_CHUNKS
#define TR_P_CHUNKS 2
#endif
  // P is published to the MMA warp in NPC key chunks (each its own barrier),
  // so O += P.V starts on the first chunk while the rest is still exponentiated
  static constexpr int NPC = TR_P_CHUNKS;
  static_assert(NPC == 2 || NPC == 4, "P chunks: 2 or 4");
};

// Per-CTA kv tile walk: the tile count of every kv segment lives in shared
// memory (no dynamically indexed local arrays), and each role advances its
// own (segment, tile) cursor.
#ifdef TR_TRACE
// Debug-only timeline of CTA 0 (clock64 per role and kv tile); read back with
// tr_debug_trace().  Not compiled into the product library.
// CTAs 0 and 1 (a pair in the TR_KERNEL_PAIR build); slots 0-5 clock64,
// slot 6-7 free; TR_TRACE_GT(slot) records %globaltimer (cross-SM).
static __device__ unsigned long long g_trace[2 * 20 * 64 * 8];   // [CTA][warp < 20][tile][slot]
#define TR_TRACE_AT(slot, jj)                                                        \
  do {                                                                               \
    if (blockIdx.x < 2 && lane == 0 && (jj) >= 0 && (jj) < 64)                                  \
      g_trace[((blockIdx.x * 20 + warp) * 64 + (jj)) * 8 + (slot)] = clock64();      \
  } while (0)
#define TR_TRACE_W(w, slot, jj)                                                      \
  do {                                                                               \
    if (blockIdx.x < 2 && lane == 0 && (jj) >= 0 && (jj) < 64)                                  \
      g_trace[((blockIdx.x * 20 + (w)) * 64 + (jj)) * 8 + (slot)] = clock64();       \
  } while (0)
#define TR_TRACE_GT(slot, jj)                                                        \
  do {                                                                               \
    if (blockIdx.x < 2 && lane == 0 && (jj) >= 0 && (jj) < 64)                                  \
      g_trace[((blockIdx.x * 20 + warp) * 64 + (jj)) * 8 + (slot)] = globaltimer_ns(); \
  } while (0)
#else
#define TR_TRACE_AT(slot, jj) \
  do {                        \
  } while (0)
#define TR_TRACE_GT(slot, jj) \
  do {                        \
  } while (0)
#define TR_TRACE_W(w, slot, jj) \
  do {                          \
  } while (0)
#endif

struct KvWalk {
  int g;
  int64_t t;
  __device__ __forceinline__ void next(const int64_t* tiles) {
    ++t;
    while (g < TR_MAX_SEGMENTS - 1 && t >= tiles[g]) { t = 0; ++g; }
  }
};

__device__ __forceinline__ KvWalk kv_begin(const int64_t* tiles) {
  KvWalk w{0, 0};
  while (w.g < TR_MAX_SEGMENTS - 1 && tiles[w.g] == 0) ++w.g;
  return w;
}

__device__ __forceinline__ void q_tile_of(const AttnPlan& p, int64_t lin, int& seg, int64_t& row0) {
  seg = 0;
  while (seg + 1 < p.nq && lin >= p.tile_prefix[seg + 1]) ++seg;
  int64_t local = lin - p.tile_prefix[seg];
  if (p.causal) local = (p.tile_prefix[seg + 1] - p.tile_prefix[seg]) - 1 - local;  // heavy first
  row0 = local * 256;
}

// This CTA's (head, q segment, first row): the explicit longest-first order
// when the host supplied one, else head-major with q_tile_of's order.
__device__ __forceinline__ void cta_tile(const AttnPlan& p, int64_t item, int& head, int& seg,
                                         int64_t& row0) {
  const int64_t nt = p.tile_prefix[p.nq];
  if (p.n_order == 0) {
    head = static_cast<int>(item / nt);
    q_tile_of(p, item % nt, seg, row0);
    return;
  }
  const int64_t G = p.head_group;
  const int64_t full = p.heads / G;          // complete head groups
  int64_t idx = item, g, hg;
  if (idx < full * G * nt) {
    g = idx / (G * nt);
    idx -= g * G * nt;
    hg = G;
  } else {
    g = full;
    idx -= full * G * nt;
    hg = p.heads - full * G;
  }
  head = static_cast<int>(g * G + idx % hg);
  int64_t lin = p.order[idx / hg];
  seg = 0;
  while (seg + 1 < p.nq && lin >= p.tile_prefix[seg + 1]) ++seg;
  row0 = (lin - p.tile_prefix[seg]) * 256;
}

// exp2 of one S row (already in registers) -> bf16 P in TMEM, row sums in
// packed accumulators; arrives on pbar[kh] after each of the NPC key chunks.
template <int POLY_MOD, bool kPoly, int NPC>
__device__ __forceinline__ void emit_p(const uint32_t (&s)[128], uint32_t tS, uint64_t c2,
                                       uint64_t nmc2, uint64_t (&lsum2)[2], uint64_t* pbar,
                                       int trace_j = -1) {
  constexpr int PAIRS = 64 / NPC;        // bf16 pairs (= TMEM columns) per chunk
#ifdef TR_TRACE
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#endif
  (void)trace_j;
  #pragma unroll
  for (int kh = 0; kh < NPC; ++kh) {
    uint32_t pk[PAIRS];
    #pragma unroll
    for (int ii = 0; ii < PAIRS; ++ii) {
      const int i = kh * PAIRS + ii;     // pair index in the row
      const int e = 2 * i;
      const uint64_t x2 = ffma2(f2pack(__uint_as_float(s[e]), __uint_as_float(s[e + 1])), c2, nmc2);
      float a, b;
      f2unpack(x2, a, b);
      uint64_t p2;
      if (kPoly && (i % POLY_MOD) == POLY_MOD - 1)
        p2 = exp2_poly2(f2pack(fmaxf(a, -126.f), fmaxf(b, -126.f)));
      else
        p2 = f2pack(ex2_approx(a), ex2_approx(b));
      lsum2[i & 1] = fadd2(lsum2[i & 1], p2);
      float pa, pb;
      f2unpack(p2, pa, pb);
      pk[ii] = pack_bf16x2(pa, pb);
    }
    if (kh < 2) TR_TRACE_AT(4 + 2 * kh, trace_j);     // chunk computed (store issued next)
    if constexpr (PAIRS == 32) tmem_st32(tS + kh * 32, pk);
    else tmem_st16(tS + kh * 16, pk);
    tc_wait_st();
    tc_fence_before();
    mbar_arrive(&pbar[kh]);
    if (kh < 2) TR_TRACE_AT(5 + 2 * kh, trace_j);     // chunk published
  }
}

// ------------------------------------------------------------------ host hooks
// 2-D bf16 tensor map over a (rows, row_elems) buffer, 64-element x box_rows
// boxes, 128-byte swizzle (attn_fwd_sm100.cu).
int make_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t row_elems,
              uint32_t box_rows = 128);
// measured alternatives of the D=128 kernel (attn_fwd_variants.cu); each
// returns TR_OK or a status, and -1 if not selected for this launch
int launch_attn_variant(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        AttnPlan& plan, int head_dim, int64_t blocks, cudaStream_t s);
int launch_attn_pair(const void* q, const void* k, const void* v, int64_t tq_total,
                     int64_t tk_total, AttnPlan& plan, cudaStream_t s);
int launch_attn_pair2(const void* q, const void* k, const void* v, int64_t tq_total,
                      int64_t tk_total, AttnPlan& plan, cudaStream_t s);

}  // namespace tr
