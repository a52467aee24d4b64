// Measured alternatives of the D=128 attention kernel, kept buildable and
// parity-tested but NOT the product path (DESIGN.md 5 has the A/B numbers):
//   attn_fwd_ps_kernel          P in shared memory, SS-mode P.V   (TR_ATTN_PSMEM=1)
//   attn_fwd_persistent_kernel  one CTA per SM walking the items   (TR_ATTN_PERSISTENT=1)
//   attn_fwd_pair_kernel        cta_group::2 CTA pairs             (build -D TR_KERNEL_PAIR)
// Selected at run time by launch_attn_variant (environment switches) from
// attn_fwd_sm100.cu's launcher, which otherwise runs the product kernel.
#include <cstdlib>

#include "attn_common.cuh"

namespace tr {

// ============================================================================
// attn_fwd_ps_kernel (D = 128): P goes to SHARED memory instead of TMEM.
//
// In attn_fwd_sm100_kernel P_h overwrites S_h's TMEM columns, so the next
// QK_h cannot be issued before P_h.V has read P_h: per half, every kv tile
// pays QK (512 tensor cycles) + softmax (~1650) + P.V (512) + barrier
// latencies back to back, a ~3300-cycle period against 2048 cycles of tensor
// work.  With P in shared memory (its own 2 x 32 KB, 128B-swizzled K-major
// like a Q tile; the P.V MMA reads A from smem, SS mode), S_h is free as soon
// as the softmax warps have loaded it into registers (s_free), so QK_h(j+1)
// runs while softmax_h(j) exponentiates, and the per-tile period becomes
// max(tensor 2048, softmax) -- the softmax of both halves now run side by
// side.  Measured with the softmax stubbed out (TR_EXP_NOSOFTMAX
// TR_EXP_PSMEM): SS-mode P.V + the P stores cost ~4 % of the pipeline's
// throughput, i.e. shared memory keeps up.
// Smem: Q 64 KB + P 64 KB + a 3-stage K/V ring (96 KB) consumed in the order
// K0 K1 V0 K2 V1 K3 V2 ...: every slot is released long before it is
// reloaded (V_j reuses K_j's slot, K_{j+2} reuses V_{j-1}'s).
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
// MMA order per tile j: QK0(j+1) QK1(j+1) | P0a.V P1a.V P0b.V P1b.V (j)
// (a/b = 64-key chunks; each chunk has its own full/free barrier so the
// softmax can refill chunk a of P while P.V still reads chunk b).
#ifndef TR_PS_SPLIT
#define TR_PS_SPLIT 0
#endif
constexpr int kPsIssuers = TR_PS_SPLIT ? 2 : 1;   // MMA issuer warps (1, or one per half)

struct PsCfg {
  static constexpr int D = 128;
  static constexpr int BOX = 128 * 64 * 2;        // 16 KB: 128 rows x 64 bf16
  static constexpr int TILE = 2 * BOX;            // 32 KB: 128 rows x 128 bf16
  static constexpr int NS = 3;                    // K/V ring stages
  static constexpr int THREADS = 384;
  static constexpr int SMEM_TILES = (2 + 2 + NS) * TILE;   // Q0 Q1 P0 P1 ring
  static constexpr int SMEM = SMEM_TILES + 1024 + 1024;
  static constexpr uint32_t IDESC_QK = idesc_bf16(128, 128, false);
  static constexpr uint32_t IDESC_PV = idesc_bf16(128, 128, true);
  static constexpr float RESCALE_LOG2 = 8.0f;
  static constexpr int POLY_MOD = TR_POLY_MOD;
};

// exp2 of 64 scores (one P chunk of a row) -> 8 swizzled 16-byte stores into
// the P tile; row sums accumulate in lsum2.
template <int POLY_MOD, bool kPoly>
__device__ __forceinline__ void p_chunk_smem(const uint32_t (&s)[128], int kh, uint64_t c2,
                                             uint64_t nmc2, uint64_t (&lsum2)[2], uint8_t* prow,
                                             int r) {
  #pragma unroll
  for (int c16 = 0; c16 < 8; ++c16) {
    uint32_t w[4];
    #pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const int i = kh * 32 + c16 * 4 + q4;     // pair index in the row
      const uint64_t x2 = ffma2(f2pack(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), c2, nmc2);
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
      w[q4] = pack_bf16x2(pa, pb);
    }
    *reinterpret_cast<uint4*>(prow + kh * PsCfg::BOX + r * 128 + ((c16 ^ (r & 7)) * 16)) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void __launch_bounds__(384, 1)
attn_fwd_ps_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                   const __grid_constant__ CUtensorMap tmv, const __grid_constant__ AttnPlan p) {
  using C = PsCfg;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                        // 2 tiles
  uint8_t* sP = smem + 2 * C::TILE;          // 2 tiles
  uint8_t* sKV = smem + 4 * C::TILE;         // NS tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_TILES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;              // [NS]
  uint64_t* kv_empty = kv_full + C::NS;      // [NS]
  uint64_t* s_full = kv_empty + C::NS;       // [2]
  uint64_t* s_free = s_full + 2;             // [2]
  uint64_t* p_full = s_free + 2;             // [2 halves][2 chunks]
  uint64_t* p_free = p_full + 4;             // [2 halves][2 chunks]
  uint64_t* o_done = p_free + 4;             // [2]
  int64_t* kv_tiles = reinterpret_cast<int64_t*>(o_done + 2);   // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_tiles + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  int head, qseg;
  int64_t qrow0;
  cta_tile(p, blockIdx.x, head, qseg, qrow0);
  const tr_segment Q = p.q[qseg];
  const int64_t qmax_pos = Q.pos0 + imin64(qrow0 + 255, Q.rows - 1);

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::NS; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], kPsIssuers); }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&s_full[h], 1);
      mbar_init(&s_free[h], 128);
      mbar_init(&o_done[h], 1);
      for (int c = 0; c < 2; ++c) {
        mbar_init(&p_full[2 * h + c], 128);
        mbar_init(&p_free[2 * h + c], 1);
      }
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmq); tma_prefetch_desc(&tmk); tma_prefetch_desc(&tmv);
  }
  if (warp == 2 && lane < TR_MAX_SEGMENTS) {
    int64_t n = 0;
    if (lane < p.nkv) {
      n = (p.kv[lane].rows + 127) / 128;
      if (p.causal)
        n = (qmax_pos < p.kv[lane].pos0) ? 0 : imin64(n, (qmax_pos - p.kv[lane].pos0) / 128 + 1);
    }
    kv_tiles[lane] = n;
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int ntiles = __shfl_sync(
      0xffffffffu, static_cast<int>(kv_tiles[0] + kv_tiles[1] + kv_tiles[2] + kv_tiles[3]), 0);

  if (warp < 4) {
   setmaxnreg_dec<56>();
   if (warp == 0 && ntiles > 0) {
    // ------------------------------------------------------------ producer
    const int32_t col0 = head * D;
    mbar_arrive_expect_tx_elect(q_full, 2 * C::TILE);
    for (int h = 0; h < 2; ++h)
      for (int b = 0; b < 2; ++b)
        tma_load_2d_elect(sQ + (h * 2 + b) * C::BOX, &tmq, q_full, col0 + 64 * b,
                          static_cast<int32_t>(Q.row0 + qrow0 + 128 * h), kEvictFirst);
    int s = 0;
    uint32_t round = 0;
    auto put = [&](const CUtensorMap* tm, int64_t krow) {
      mbar_wait(&kv_empty[s], (round & 1) ^ 1);
      mbar_arrive_expect_tx_elect(&kv_full[s], C::TILE);
      for (int b = 0; b < 2; ++b)
        tma_load_2d_elect(sKV + s * C::TILE + b * C::BOX, tm, &kv_full[s], col0 + 64 * b,
                          static_cast<int32_t>(krow), kEvictLast);
      if (++s == C::NS) { s = 0; ++round; }
    };
    // consumption order: K0 K1 V0 K2 V1 K3 V2 ...
    KvWalk wk = kv_begin(kv_tiles), wv = wk;
    put(&tmk, p.kv[wk.g].row0 + wk.t * 128);                 // K0
    wk.next(kv_tiles);
    if (ntiles > 1) {
      put(&tmk, p.kv[wk.g].row0 + wk.t * 128);               // K1
      wk.next(kv_tiles);
    }
    for (int j = 0; j < ntiles; ++j) {
      put(&tmv, p.kv[wv.g].row0 + wv.t * 128);               // V_j
      wv.next(kv_tiles);
      if (j + 2 < ntiles) {
        put(&tmk, p.kv[wk.g].row0 + wk.t * 128);             // K_{j+2}
        wk.next(kv_tiles);
      }
    }
   } else if ((warp == 1 || (kPsIssuers == 2 && warp == 3)) && ntiles > 0) {
    // ------------------------------------------------------------ MMA issuer(s)
    const uint64_t dQ = sdesc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t dP = sdesc_sw128(smem_u32(sP), 16, 1024);
    const uint64_t dK = sdesc_sw128(smem_u32(sKV), 16, 1024);
    const uint64_t dV = sdesc_sw128(smem_u32(sKV), C::BOX, 1024);
    int n_idx = 0;
    auto take = [&]() {
      const int slot = n_idx % C::NS;
      mbar_wait(&kv_full[slot], static_cast<uint32_t>((n_idx / C::NS) & 1));
      tc_fence_after();
      ++n_idx;
      return slot;
    };
    auto qk = [&](int h, int slot) {
      const uint64_t a0 = dQ + static_cast<uint32_t>((h * C::TILE) >> 4);
      const uint64_t b0 = dK + static_cast<uint32_t>((slot * C::TILE) >> 4);
      #pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = ((kk / 4) * C::BOX + (kk % 4) * 32) >> 4;
        mma_ss_elect(tmem + h * 128, desc_add(a0, off), desc_add(b0, off), C::IDESC_QK, kk > 0);
      }
    };
    // O_h += P_h[:, chunk c keys] . V[chunk c keys, :]   (A from smem)
    auto pv = [&](int h, int slot, int c, bool acc) {
      const uint64_t a0 = dP + static_cast<uint32_t>((h * C::TILE) >> 4);
      const uint64_t b0 = dV + static_cast<uint32_t>((slot * C::TILE) >> 4);
      #pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const int kk = c * 4 + k4;
        const uint32_t offa = ((kk / 4) * C::BOX + (kk % 4) * 32) >> 4;
        mma_ss_elect(tmem + 256 + h * 128, desc_add(a0, offa), desc_add(b0, (kk * 2048) >> 4),
                     C::IDESC_PV, (acc || k4 > 0) ? 1u : 0u);
      }
    };
    mbar_wait(q_full, 0);
    tc_fence_after();
    if constexpr (kPsIssuers == 2) {
      // one issuer per half (warp 1: half 0, warp 3: half 1), each in its own
      // half's natural order; half 1 starts once half 0 has published its
      // first P chunk, so the two softmax groups run staggered (one
      // exponentiates while the other loads S / reduces its max)
      const int h = (warp == 1) ? 0 : 1;
      int ks = take();                                        // K0
      if (h == 1) mbar_wait(&p_full[0], 0);
      qk(h, ks);
      tc_commit_elect(&s_full[h]);
      tc_commit_elect(&kv_empty[ks]);
      for (int j = 0; j < ntiles; ++j) {
        const uint32_t ph = j & 1;
        if (j + 1 < ntiles) {
          ks = take();                                        // K_{j+1}
          mbar_wait(&s_free[h], ph);
          tc_fence_after();
          qk(h, ks);
          tc_commit_elect(&s_full[h]);
          tc_commit_elect(&kv_empty[ks]);
        }
        const int vs = take();                                // V_j
        #pragma unroll
        for (int c = 0; c < 2; ++c) {
          mbar_wait(&p_full[2 * h + c], ph);
          tc_fence_after();
          pv(h, vs, c, j > 0 || c > 0);
          tc_commit_elect(&p_free[2 * h + c]);
        }
        tc_commit_elect(&kv_empty[vs]);
      }
      tc_commit_elect(&o_done[h]);
    } else {
      int ks = take();                                          // K0
      qk(0, ks);
      tc_commit_elect(&s_full[0]);
      qk(1, ks);
      tc_commit_elect(&s_full[1]);
      tc_commit_elect(&kv_empty[ks]);
      for (int j = 0; j < ntiles; ++j) {
        const uint32_t ph = j & 1;
        TR_TRACE_AT(0, j);
        if (j + 1 < ntiles) {
          ks = take();                                          // K_{j+1}
          mbar_wait(&s_free[0], ph);
          tc_fence_after();
          qk(0, ks);
          tc_commit_elect(&s_full[0]);
          mbar_wait(&s_free[1], ph);
          tc_fence_after();
          qk(1, ks);
          tc_commit_elect(&s_full[1]);
          tc_commit_elect(&kv_empty[ks]);
        }
        TR_TRACE_AT(1, j);
        const int vs = take();                                  // V_j
        TR_TRACE_AT(2, j);
        #pragma unroll
        for (int c = 0; c < 2; ++c) {
          #pragma unroll
          for (int h = 0; h < 2; ++h) {
            mbar_wait(&p_full[2 * h + c], ph);
            tc_fence_after();
            pv(h, vs, c, j > 0 || c > 0);
            tc_commit_elect(&p_free[2 * h + c]);
          }
        }
        tc_commit_elect(&kv_empty[vs]);
        TR_TRACE_AT(3, j);
      }
      tc_commit_elect(&o_done[0]);
      tc_commit_elect(&o_done[1]);
    }
   }
  } else {
   setmaxnreg_inc<224>();
   {
    // ------------------------------------------------------------ softmax + epilogue
    const int h = (warp - 4) / 4;
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + h * 128;
    const uint32_t tO = tmem + lane_base + 256 + h * 128;
    uint8_t* prow = sP + h * C::TILE;
    const int64_t row_in_seg = qrow0 + 128 * h + r;
    const int64_t my_pos = Q.pos0 + row_in_seg;
    const int64_t half_min_pos = Q.pos0 + qrow0 + 128 * h;
    const float c = p.scale_log2;
    const float thresh = C::RESCALE_LOG2 / c;
    const uint64_t c2 = f2pack(c, c);
    float m_used = -INFINITY;
    uint64_t lsum2[2] = {0ull, 0ull};
    KvWalk w = kv_begin(kv_tiles);
    for (int j = 0; j < ntiles; ++j, w.next(kv_tiles)) {
      const uint32_t ph = j & 1;
      const int64_t kpos = p.kv[w.g].pos0 + w.t * 128;
      const int valid = static_cast<int>(imin64(128, p.kv[w.g].rows - w.t * 128));
      TR_TRACE_AT(0, j);
      mbar_wait(&s_full[h], ph);
      tc_fence_after();
      TR_TRACE_AT(1, j);
      uint32_t s[128];
      tmem_ld32_at<0>(tS + 0, s);
      tmem_ld32_at<32>(tS + 32, s);
      tmem_ld32_at<64>(tS + 64, s);
      tmem_ld32_at<96>(tS + 96, s);
      tc_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_free[h]);            // S_h may now be overwritten by QK_h(j+1)
      const bool need_mask = valid < 128 || (p.causal && kpos + 127 > half_min_pos);
      if (need_mask) {
        int64_t lim = valid;
        if (p.causal) lim = imin64(lim, my_pos - kpos + 1);
        const int limit = static_cast<int>(imax64(lim, 0));
        #pragma unroll
        for (int i = 0; i < 128; ++i) s[i] = (i < limit) ? s[i] : 0xFF800000u;
      }
      float mx = __uint_as_float(s[0]);
      float mxb = __uint_as_float(s[1]);
      #pragma unroll
      for (int i = 2; i < 128; i += 4) {
        mx = fmaxf(mx, fmaxf(__uint_as_float(s[i]), __uint_as_float(s[i + 1])));
        mxb = fmaxf(mxb, fmaxf(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3])));
      }
      mx = fmaxf(mx, mxb);
      TR_TRACE_AT(2, j);
      const bool grow = mx > m_used + thresh;
      const bool scale_o = grow && m_used != -INFINITY;
      if (__any_sync(0xffffffffu, scale_o)) {
        // O_h must hold every P.V of earlier tiles: wait for the last chunk
        // of P_h(j-1).V (the chunks complete in order)
        mbar_wait(&p_free[2 * h + 1], ph ^ 1);
        tc_fence_after();
        const float f = scale_o ? ex2_approx((m_used - mx) * c) : 1.f;
        const uint64_t f2 = f2pack(f, f);
        lsum2[0] = fmul2(lsum2[0], f2);
        lsum2[1] = fmul2(lsum2[1], f2);
        #pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t u[32];
          tmem_ld32(tO + cc * 32, u);
          tc_wait_ld();
          #pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t v = fmul2(f2pack(__uint_as_float(u[i]), __uint_as_float(u[i + 1])), f2);
            u[i] = static_cast<uint32_t>(v);
            u[i + 1] = static_cast<uint32_t>(v >> 32);
          }
          tmem_st32(tO + cc * 32, u);
        }
        tc_wait_st();
      }
      if (grow) m_used = mx;
      const float mc = (m_used == -INFINITY) ? 0.f : m_used * c;
      const uint64_t nmc2 = f2pack(-mc, -mc);
      #pragma unroll
      for (int kh = 0; kh < 2; ++kh) {
        // P_h(j-1).V has finished reading this chunk of the P tile
        mbar_wait(&p_free[2 * h + kh], ph ^ 1);
        TR_TRACE_AT(3 + 2 * kh, j);
        if (need_mask)
          p_chunk_smem<C::POLY_MOD, false>(s, kh, c2, nmc2, lsum2, prow, r);
        else
          p_chunk_smem<C::POLY_MOD, true>(s, kh, c2, nmc2, lsum2, prow, r);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&p_full[2 * h + kh]);
        TR_TRACE_AT(4 + 2 * kh, j);
      }
    }
    float l;
    {
      float a0, a1, b0, b1;
      f2unpack(lsum2[0], a0, a1);
      f2unpack(lsum2[1], b0, b1);
      l = (a0 + a1) + (b0 + b1);
    }
    // ---------------------------------------------------------- epilogue
    const bool row_ok = row_in_seg < Q.rows;
    const int64_t grow = Q.row0 + row_in_seg;
    const int64_t oidx = (grow * p.heads + head) * D;
    if (ntiles > 0) {
      mbar_wait(&o_done[h], 0);
      tc_fence_after();
    }
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    #pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t u[32];
      if (ntiles > 0) {
        tmem_ld32(tO + cc * 32, u);
        tc_wait_ld();
      } else {
        #pragma unroll
        for (int i = 0; i < 32; ++i) u[i] = 0u;
      }
      if (p.out_f32) {
        if (row_ok) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + oidx + cc * 32);
          #pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(u[4 * i]) * inv, __uint_as_float(u[4 * i + 1]) * inv,
                                 __uint_as_float(u[4 * i + 2]) * inv, __uint_as_float(u[4 * i + 3]) * inv);
        }
        continue;
      }
      uint32_t pk[16];
      #pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = pack_bf16x2(__uint_as_float(u[2 * i]) * inv, __uint_as_float(u[2 * i + 1]) * inv);
      if (row_ok) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + oidx + cc * 32);
        #pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (row_ok)
      p.lse[head * p.lse_stride + grow] = (l > 0.f) ? (logf(l) + m_used * p.scale) : -INFINITY;
   }
  }
  tc_fence_before();
  if (p.done_flag) __threadfence_system();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (p.done_flag && threadIdx.x == 0) signal_done(p);
}

// ============================================================================
// Persistent form of attn_fwd_sm100_kernel: one CTA per SM walks the work
// items (head x 256-row q tile, in the same order as the one-CTA-per-item
// grid) with a static stride of gridDim.x.  Barrier initialisation, the TMEM
// allocation and the tensor-map prefetch happen once per SM instead of once
// per item, and consecutive items overlap: the producer loads the next
// item's Q (as soon as the last QK of the current item has read the Q tile)
// and K/V into the ring while the current item drains, the next item's first
// QK MMAs run while the softmax warps are still in the current item's
// epilogue, and the epilogue releases O right after reading it (o_free) so
// the next P.V can overwrite it.  Every barrier phase is tracked across
// items: per-tile barriers by a running tile count, per-item barriers by a
// running count of items that have kv tiles.
template <int D>
__device__ __forceinline__ int item_kv_tiles(const AttnPlan& p, int64_t qmax_pos, int lane,
                                             int64_t* my_tiles) {
  // this warp's copy of the item's per-kv-segment tile counts
  if (lane < TR_MAX_SEGMENTS) {
    int64_t n = 0;
    if (lane < p.nkv) {
      n = (p.kv[lane].rows + 127) / 128;
      if (p.causal)
        n = (qmax_pos < p.kv[lane].pos0) ? 0 : imin64(n, (qmax_pos - p.kv[lane].pos0) / 128 + 1);
    }
    my_tiles[lane] = n;
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu,
                     static_cast<int>(my_tiles[0] + my_tiles[1] + my_tiles[2] + my_tiles[3]), 0);
}

template <int D>
__global__ void __launch_bounds__(384, 1)
attn_fwd_persistent_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                           const __grid_constant__ CUtensorMap tmv, const __grid_constant__ AttnPlan p) {
  using C = AttnCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                      // 2 tiles
  uint8_t* sKV = smem + 2 * C::TILE;       // NS tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_TILES);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;                 // [NS]
  uint64_t* kv_empty = kv_full + C::NS;         // [NS]
  uint64_t* s_full = kv_empty + C::NS;          // [2]
  uint64_t* p_full = s_full + 2;                // [2 halves][NPC key chunks]
  uint64_t* o_done = p_full + 2 * C::NPC;       // [2]
  uint64_t* o_free = o_done + 2;                // [2]
  int64_t* kv_tiles = reinterpret_cast<int64_t*>(o_free + 2);   // [12 warps][4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_tiles + 12 * 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  int64_t* my_tiles = kv_tiles + warp * 4;
  const int64_t n_items = p.tile_prefix[p.nq] * p.heads;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < C::NS; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&s_full[h], 1);
      for (int kh = 0; kh < C::NPC; ++kh) mbar_init(&p_full[C::NPC * h + kh], 128);
      mbar_init(&o_done[h], 1);
      mbar_init(&o_free[h], 128);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmq); tma_prefetch_desc(&tmk); tma_prefetch_desc(&tmv);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  if (warp < 4) {
   setmaxnreg_dec<56>();
   if (warp == 0) {
    // ------------------------------------------------------------ producer
    int s = 0;
    uint32_t round = 0, act = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      int head, qseg;
      int64_t qrow0;
      cta_tile(p, item, head, qseg, qrow0);
      const tr_segment Q = p.q[qseg];
      const int64_t qmax_pos = Q.pos0 + imin64(qrow0 + 255, Q.rows - 1);
      const int ntiles = item_kv_tiles<D>(p, qmax_pos, lane, my_tiles);
      if (ntiles == 0) continue;
      const int32_t col0 = head * D;
      mbar_wait(q_empty, (act & 1) ^ 1);     // the previous item's QKs have read sQ
      mbar_arrive_expect_tx_elect(q_full, 2 * C::TILE);
      for (int h = 0; h < 2; ++h)
        for (int b = 0; b < C::NB; ++b)
          tma_load_2d_elect(sQ + (h * C::NB + b) * C::BOX, &tmq, q_full, col0 + 64 * b,
                            static_cast<int32_t>(Q.row0 + qrow0 + 128 * h), kEvictFirst);
      KvWalk w = kv_begin(my_tiles);
      for (int j = 0; j < ntiles; ++j, w.next(my_tiles)) {
        const int32_t krow = static_cast<int32_t>(p.kv[w.g].row0 + w.t * 128);
        #pragma unroll
        for (int which = 0; which < 2; ++which) {
          mbar_wait(&kv_empty[s], (round & 1) ^ 1);
          mbar_arrive_expect_tx_elect(&kv_full[s], C::TILE);
          const CUtensorMap* tm = which ? &tmv : &tmk;
          #pragma unroll
          for (int b = 0; b < C::NB; ++b)
            tma_load_2d_elect(sKV + s * C::TILE + b * C::BOX, tm, &kv_full[s], col0 + 64 * b, krow,
                              kEvictLast);
          if (++s == C::NS) { s = 0; ++round; }
        }
      }
      ++act;
    }
   } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t q_addr = smem_u32(sQ);
    const uint32_t kv_addr = smem_u32(sKV);
    const uint64_t dK = sdesc_sw128(kv_addr, 16, 1024);
    const uint64_t dQ = sdesc_sw128(q_addr, 16, 1024);
    const uint64_t dV = sdesc_sw128(kv_addr, C::BOX, 1024);
    auto qk = [&](int h, int stage) {
      const uint64_t a0 = dQ + static_cast<uint32_t>((h * C::TILE) >> 4);
      const uint64_t b0 = dK + static_cast<uint32_t>((stage * C::TILE) >> 4);
      #pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = ((kk / 4) * C::BOX + (kk % 4) * 32) >> 4;
        mma_ss_elect(tmem + h * 128, desc_add(a0, off), desc_add(b0, off), C::IDESC_QK, kk > 0);
      }
    };
    constexpr int KPC = 8 / C::NPC;
    auto pv = [&](int h, int stage, int kh, bool acc) {
      const uint64_t b0 = dV + static_cast<uint32_t>((stage * C::TILE) >> 4);
      #pragma unroll
      for (int k4 = 0; k4 < KPC; ++k4) {
        const int kk = kh * KPC + k4;
        mma_ts_elect(tmem + 256 + h * 128, tmem + h * 128 + kk * 8, desc_add(b0, (kk * 2048) >> 4),
                     C::IDESC_PV, (acc || kk > 0) ? 1u : 0u);
      }
    };
    uint32_t act = 0;
    uint64_t T = 0;                       // kv tiles of earlier items (per-tile phases)
    // O_h of the previous item must have been read by its epilogue before the
    // first (non-accumulating) P.V of this item overwrites it
    auto pv_both = [&](int h, int stage, uint64_t tile, bool acc) {
      if (!acc) {
        mbar_wait(&o_free[h], (act & 1) ^ 1);
        tc_fence_after();
      }
      #pragma unroll
      for (int kh = 0; kh < C::NPC; ++kh) {
        mbar_wait(&p_full[C::NPC * h + kh], static_cast<uint32_t>(tile & 1));
        tc_fence_after();
        pv(h, stage, kh, acc || kh > 0);
      }
    };
    int sk = 0;
    uint32_t rk = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      int head, qseg;
      int64_t qrow0;
      cta_tile(p, item, head, qseg, qrow0);
      const tr_segment Q = p.q[qseg];
      const int64_t qmax_pos = Q.pos0 + imin64(qrow0 + 255, Q.rows - 1);
      const int ntiles = item_kv_tiles<D>(p, qmax_pos, lane, my_tiles);
      if (ntiles == 0) continue;
      mbar_wait(q_full, act & 1);
      tc_fence_after();
      int prev_v_stage = 0;
      for (int j = 0; j < ntiles; ++j) {
        const int sv = (sk + 1 == C::NS) ? 0 : sk + 1;
        const uint32_t rv = (sk + 1 == C::NS) ? rk + 1 : rk;
        mbar_wait(&kv_full[sk], rk & 1);
        tc_fence_after();
        qk(0, sk);
        tc_commit_elect(&s_full[0]);
        if (j > 0) {
          pv_both(1, prev_v_stage, T + j - 1, j - 1 > 0);
          tc_commit_elect(&kv_empty[prev_v_stage]);
        }
        qk(1, sk);
        tc_commit_elect(&s_full[1]);
        tc_commit_elect(&kv_empty[sk]);
        if (j == ntiles - 1) tc_commit_elect(q_empty);   // sQ free for the next item
        mbar_wait(&kv_full[sv], rv & 1);
        pv_both(0, sv, T + j, j > 0);
        if (j == ntiles - 1) tc_commit_elect(&o_done[0]);
        prev_v_stage = sv;
        sk = (sv + 1 == C::NS) ? 0 : sv + 1;
        rk = (sv + 1 == C::NS) ? rv + 1 : rv;
      }
      pv_both(1, prev_v_stage, T + ntiles - 1, ntiles - 1 > 0);
      tc_commit_elect(&kv_empty[prev_v_stage]);
      tc_commit_elect(&o_done[1]);
      T += ntiles;
      ++act;
    }
   }
  } else {
   setmaxnreg_inc<224>();
   {
    // ------------------------------------------------------------ softmax + epilogue
    const int h = (warp - 4) / 4;
    const int quarter = warp % 4;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + h * 128;
    const uint32_t tO = tmem + lane_base + 256 + h * 128;
    const float c = p.scale_log2;
    const float thresh = C::RESCALE_LOG2 / c;
    const uint64_t c2 = f2pack(c, c);
    uint32_t act = 0;
    uint64_t T = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      int head, qseg;
      int64_t qrow0;
      cta_tile(p, item, head, qseg, qrow0);
      const tr_segment Q = p.q[qseg];
      const int64_t qmax_pos = Q.pos0 + imin64(qrow0 + 255, Q.rows - 1);
      const int ntiles = item_kv_tiles<D>(p, qmax_pos, lane, my_tiles);
      const int64_t row_in_seg = qrow0 + 128 * h + r;
      const int64_t my_pos = Q.pos0 + row_in_seg;
      const int64_t half_min_pos = Q.pos0 + qrow0 + 128 * h;
      float m_used = -INFINITY;
      uint64_t lsum2[2] = {0ull, 0ull};
      KvWalk w = kv_begin(my_tiles);
      for (int j = 0; j < ntiles; ++j, w.next(my_tiles)) {
        const int64_t kpos = p.kv[w.g].pos0 + w.t * 128;
        const int valid = static_cast<int>(imin64(128, p.kv[w.g].rows - w.t * 128));
        mbar_wait(&s_full[h], static_cast<uint32_t>((T + j) & 1));
        tc_fence_after();
        uint32_t s[128];
        tmem_ld32_at<0>(tS + 0, s);
        tmem_ld32_at<32>(tS + 32, s);
        tmem_ld32_at<64>(tS + 64, s);
        tmem_ld32_at<96>(tS + 96, s);
        tc_wait_ld();
        const bool need_mask = valid < 128 || (p.causal && kpos + 127 > half_min_pos);
        if (need_mask) {
          int64_t lim = valid;
          if (p.causal) lim = imin64(lim, my_pos - kpos + 1);
          const int limit = static_cast<int>(imax64(lim, 0));
          #pragma unroll
          for (int i = 0; i < 128; ++i) s[i] = (i < limit) ? s[i] : 0xFF800000u;
        }
        float mx = __uint_as_float(s[0]);
        float mxb = __uint_as_float(s[1]);
        #pragma unroll
        for (int i = 2; i < 128; i += 4) {
          mx = fmaxf(mx, fmaxf(__uint_as_float(s[i]), __uint_as_float(s[i + 1])));
          mxb = fmaxf(mxb, fmaxf(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3])));
        }
        mx = fmaxf(mx, mxb);
        const bool grow = mx > m_used + thresh;
        const bool scale_o = grow && m_used != -INFINITY;
        if (__any_sync(0xffffffffu, scale_o)) {
          // this tile's S commit implies every earlier MMA (this item's P.V
          // products included) has completed: O is quiescent
          const float f = scale_o ? ex2_approx((m_used - mx) * c) : 1.f;
          const uint64_t f2 = f2pack(f, f);
          lsum2[0] = fmul2(lsum2[0], f2);
          lsum2[1] = fmul2(lsum2[1], f2);
          #pragma unroll
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t u[32];
            tmem_ld32(tO + cc * 32, u);
            tc_wait_ld();
            #pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const uint64_t v = fmul2(f2pack(__uint_as_float(u[i]), __uint_as_float(u[i + 1])), f2);
              u[i] = static_cast<uint32_t>(v);
              u[i + 1] = static_cast<uint32_t>(v >> 32);
            }
            tmem_st32(tO + cc * 32, u);
          }
        }
        if (grow) m_used = mx;
        const float mc = (m_used == -INFINITY) ? 0.f : m_used * c;
        const uint64_t nmc2 = f2pack(-mc, -mc);
        if (need_mask)
          emit_p<C::POLY_MOD, false, C::NPC>(s, tS, c2, nmc2, lsum2, &p_full[C::NPC * h]);
        else
          emit_p<C::POLY_MOD, true, C::NPC>(s, tS, c2, nmc2, lsum2, &p_full[C::NPC * h]);
      }
      float l;
      {
        float a0, a1, b0, b1;
        f2unpack(lsum2[0], a0, a1);
        f2unpack(lsum2[1], b0, b1);
        l = (a0 + a1) + (b0 + b1);
      }
      // ---------------------------------------------------------- epilogue
      const bool row_ok = row_in_seg < Q.rows;
      const int64_t grow = Q.row0 + row_in_seg;
      const int64_t oidx = (grow * p.heads + head) * D;
      const float inv = (l > 0.f) ? 1.f / l : 0.f;
      uint32_t u[D];
      if (ntiles > 0) {
        mbar_wait(&o_done[h], act & 1);
        tc_fence_after();
        tmem_ld32_at<0>(tO, u);
        tmem_ld32_at<32>(tO + 32, u);
        if constexpr (D == 128) {
          tmem_ld32_at<64>(tO + 64, u);
          tmem_ld32_at<96>(tO + 96, u);
        }
        tc_wait_ld();
        tc_fence_before();
        mbar_arrive(&o_free[h]);          // the next item's P.V may overwrite O_h
      } else {
        #pragma unroll
        for (int i = 0; i < D; ++i) u[i] = 0u;
      }
      if (row_ok) {
        if (p.out_f32) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + oidx);
          #pragma unroll
          for (int i = 0; i < D / 4; ++i)
            dst[i] = make_float4(__uint_as_float(u[4 * i]) * inv, __uint_as_float(u[4 * i + 1]) * inv,
                                 __uint_as_float(u[4 * i + 2]) * inv, __uint_as_float(u[4 * i + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + oidx);
          #pragma unroll
          for (int i = 0; i < D / 8; ++i)
            dst[i] = make_uint4(pack_bf16x2(__uint_as_float(u[8 * i]) * inv, __uint_as_float(u[8 * i + 1]) * inv),
                                pack_bf16x2(__uint_as_float(u[8 * i + 2]) * inv, __uint_as_float(u[8 * i + 3]) * inv),
                                pack_bf16x2(__uint_as_float(u[8 * i + 4]) * inv, __uint_as_float(u[8 * i + 5]) * inv),
                                pack_bf16x2(__uint_as_float(u[8 * i + 6]) * inv, __uint_as_float(u[8 * i + 7]) * inv));
        }
        p.lse[head * p.lse_stride + grow] = (l > 0.f) ? (logf(l) + m_used * p.scale) : -INFINITY;
      }
      T += ntiles;
      if (ntiles > 0) ++act;
    }
   }
  }
  tc_fence_before();
  if (p.done_flag) __threadfence_system();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (p.done_flag && threadIdx.x == 0) signal_done(p);
}

#ifdef TR_KERNEL_PAIR
// Opt-in build variant (python -m paper_2412_20501_b200.build -D TR_KERNEL_PAIR):
// parity-green, faster in short bursts, slower than attn_fwd_sm100_kernel under
// the 1000 W power cap.  Not compiled into the product library.
// exp2 of 64 scores -> 32 packed bf16x2 words of P; row-sum in lsum2.
template <int POLY_MOD, bool kPoly>
__device__ __forceinline__ void p_row64(const uint32_t (&s)[64], uint64_t c2, uint64_t nmc2,
                                        uint64_t (&lsum2)[2], uint32_t (&pk)[32]) {
  #pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint64_t x2 =
        ffma2(f2pack(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), c2, nmc2);
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
    pk[i] = pack_bf16x2(pa, pb);
  }
}

// ============================================================================
// attn_fwd_pair: the D=128 kernel.  A CTA PAIR (cluster of 2 on one TPC)
// computes one head x 256 query rows with cta_group::2 MMAs (M=256): CTA r
// holds q rows [128r, 128r+128) and HALF of every K tile (keys 64r..64r+63)
// and V tile (head-dim columns 64r..64r+63), so each SM streams the same
// K/V bytes per flop as a 256-row CTA while its TMEM holds only one 128-row
// tile -- room for DOUBLE-BUFFERED S:
//   TMEM (512 cols, same columns in both CTAs): S_buf at buf*128,
//   O_A at 256, O_B at 384.
// The softmax of each CTA is split by KEY COLUMNS over its 8 warps into two
// independent online softmaxes (group g owns keys 64g..64g+63 of every tile
// and accumulates O_g); the two are merged row by row in the epilogue.
// Leader (rank 0) MMA order:  S(0) S(1) | per j: O_A+=P_A(j)V_j[keys 0:64]
//                                               O_B+=P_B(j)V_j[keys 64:128]
//                                               S(j+2) -> buffer j&1
// so S(j+1) is in TMEM while softmax(j) runs: the P -> P.V -> next-S chain is
// off the critical path.  K/V halves cross each CTA's ring in consumption
// order K0 K1 V0 K2 V1 ...; TMA completions count on the leader's barriers,
// MMA completions are multicast to both CTAs, P hand-offs arrive (one per
// warp) on the leader's barriers.
#ifdef TR_PAIR_SLEEP_NS
#define PAIR_WAIT(bar, par) mbar_wait_backoff(bar, par, TR_PAIR_SLEEP_NS)
#else
#define PAIR_WAIT(bar, par) mbar_wait_cluster(bar, par)
#endif
struct PairCfg {
  static constexpr int D = 128;
  static constexpr int QBOX = 128 * 64 * 2;       // q tile box: 128 rows x 64 cols
  static constexpr int QTILE = 2 * QBOX;          // this CTA's 128 q rows (32 KB)
  static constexpr int KBOX = 64 * 64 * 2;        // K half box: 64 keys x 64 cols
  static constexpr int STAGE = 16384;             // K half (2 x KBOX) or V half (128 x 64)
  static constexpr int NS = 12;                   // ring stages
  static constexpr int THREADS = 384;
  static constexpr int SMEM_TILES = QTILE + NS * STAGE;
  static constexpr int SMEM = SMEM_TILES + 1024 /*barriers*/ + 1024 /*alignment slack*/;
  static constexpr uint32_t IDESC_QK = idesc_bf16(256, 128, false);
  static constexpr uint32_t IDESC_PV = idesc_bf16(256, 128, true);
  static constexpr float RESCALE_LOG2 = 8.0f;
  static constexpr int POLY_MOD = TR_POLY_MOD;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk64,
                     const __grid_constant__ CUtensorMap tmv, const __grid_constant__ AttnPlan p) {
  using C = PairCfg;
  constexpr int D = C::D;
#ifndef TR_PAIR_MMA_WARP
#define TR_PAIR_MMA_WARP 1
#define TR_PAIR_PROD_WARP 0
#endif
  constexpr int kMmaWarp = TR_PAIR_MMA_WARP, kProdWarp = TR_PAIR_PROD_WARP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + C::QTILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_TILES);
  uint64_t* q_full = bars + 0;               // leader: both q halves landed
  uint64_t* kv_full = bars + 1;              // [NS] leader: both halves of a stage landed
  uint64_t* kv_empty = kv_full + C::NS;      // [NS] both CTAs (multicast commit)
  uint64_t* s_full = kv_empty + C::NS;       // [2 buffers] both CTAs
  uint64_t* p_full = s_full + 2;             // [2 buffers][2 groups] leader, 8 warp arrivals
  uint64_t* pv_done = p_full + 4;            // [2 groups] both CTAs
  uint64_t* o_done = pv_done + 2;            // [1] both CTAs
  int64_t* kv_tiles = reinterpret_cast<int64_t*>(o_done + 1);   // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 5);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int64_t pair = blockIdx.x >> 1;
  const int head = static_cast<int>(pair / p.tile_prefix[p.nq]);
  const int64_t lin = pair % p.tile_prefix[p.nq];
  int qseg;
  int64_t qrow0;                             // first row of the pair's 256-row tile
  q_tile_of(p, lin, qseg, qrow0);
  const tr_segment Q = p.q[qseg];
  const int64_t qmax_pos = Q.pos0 + imin64(qrow0 + 255, Q.rows - 1);
  const int64_t my_row0 = qrow0 + 128 * rank;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::NS; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int b = 0; b < 2; ++b) mbar_init(&s_full[b], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&p_full[i], 8);
    for (int g = 0; g < 2; ++g) mbar_init(&pv_done[g], 1);
    mbar_init(o_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmq); tma_prefetch_desc(&tmk64); tma_prefetch_desc(&tmv);
  }
  if (warp == 2 && lane < TR_MAX_SEGMENTS) {
    int64_t n = 0;
    if (lane < p.nkv) {
      n = (p.kv[lane].rows + 127) / 128;
      if (p.causal)
        n = (qmax_pos < p.kv[lane].pos0) ? 0 : imin64(n, (qmax_pos - p.kv[lane].pos0) / 128 + 1);
    }
    kv_tiles[lane] = n;
  }
  if (warp == kMmaWarp) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();                            // peer barriers initialised before any remote use
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int ntiles = __shfl_sync(
      0xffffffffu, static_cast<int>(kv_tiles[0] + kv_tiles[1] + kv_tiles[2] + kv_tiles[3]), 0);

  if (warp < 4) {
   setmaxnreg_dec<56>();
   if (warp == kProdWarp && ntiles > 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    const int32_t col0 = head * D;
    const uint32_t lq_full = mapa_u32(smem_u32(q_full), 0);
    if (rank == 0) mbar_arrive_expect_tx_elect(q_full, 2 * C::QTILE);
    for (int b = 0; b < 2; ++b)
      tma_load_2d_pair_elect(sQ + b * C::QBOX, &tmq, lq_full, col0 + 64 * b,
                             static_cast<int32_t>(Q.row0 + my_row0), kEvictFirst);
    int s = 0;
    uint32_t round = 0;
    auto put = [&](bool is_v, int64_t krow) {
      PAIR_WAIT(&kv_empty[s], (round & 1) ^ 1);
      if (rank == 0) mbar_arrive_expect_tx_elect(&kv_full[s], 2 * C::STAGE);
      const uint32_t lbar = mapa_u32(smem_u32(&kv_full[s]), 0);
      uint8_t* dst = sKV + s * C::STAGE;
      if (is_v) {          // V half: keys krow..+127, head-dim columns 64*rank..+63
        tma_load_2d_pair_elect(dst, &tmv, lbar, col0 + 64 * static_cast<int32_t>(rank),
                               static_cast<int32_t>(krow), kEvictLast);
      } else {             // K half: keys krow+64*rank..+63, all 128 head-dim columns
        for (int b = 0; b < 2; ++b)
          tma_load_2d_pair_elect(dst + b * C::KBOX, &tmk64, lbar, col0 + 64 * b,
                                 static_cast<int32_t>(krow + 64 * rank), kEvictLast);
      }
      if (++s == C::NS) { s = 0; ++round; }
    };
    KvWalk wk = kv_begin(kv_tiles), wv = wk;
    put(false, p.kv[wk.g].row0 + wk.t * 128);                        // K_0
    wk.next(kv_tiles);
    for (int j = 0; j < ntiles; ++j) {
      if (j + 1 < ntiles) {                                           // K_{j+1}
        put(false, p.kv[wk.g].row0 + wk.t * 128);
        wk.next(kv_tiles);
      }
      put(true, p.kv[wv.g].row0 + wv.t * 128);                        // V_j
      wv.next(kv_tiles);
    }
   } else if (warp == kMmaWarp && rank == 0 && ntiles > 0) {
    // ------------------------------------------------------------ MMA issuer (leader)
    mbar_wait(q_full, 0);
    tc_fence_after();
    const uint64_t dQ = sdesc_sw128(smem_u32(sQ), 16, 1024);
    const uint64_t dK = sdesc_sw128(smem_u32(sKV), 16, 1024);       // K-major
    const uint64_t dV = sdesc_sw128(smem_u32(sKV), C::STAGE, 1024); // MN-major, 64 cols / CTA
    int s = 0;
    uint32_t round = 0;
    auto take = [&]() {
      mbar_wait(&kv_full[s], round & 1);
      tc_fence_after();
      const int slot = s;
      if (++s == C::NS) { s = 0; ++round; }
      return slot;
    };
    auto qk = [&](int buf, int slot) {
      const uint64_t b0 = dK + static_cast<uint32_t>((slot * C::STAGE) >> 4);
      #pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t oa = ((kk / 4) * C::QBOX + (kk % 4) * 32) >> 4;
        const uint32_t ob = ((kk / 4) * C::KBOX + (kk % 4) * 32) >> 4;
        mma2_ss_elect(tmem + buf * 128, desc_add(dQ, oa), desc_add(b0, ob), C::IDESC_QK, kk > 0);
      }
    };
    auto pv = [&](int buf, int g, int slot, bool acc) {
      const uint64_t b0 = dV + static_cast<uint32_t>((slot * C::STAGE) >> 4);
      #pragma unroll
      for (int k4 = 0; k4 < 4; ++k4)
        mma2_ts_elect(tmem + 256 + g * 128, tmem + buf * 128 + 64 * g + 8 * k4,
                      desc_add(b0, ((g * 4 + k4) * 2048) >> 4), C::IDESC_PV,
                      (acc || k4 > 0) ? 1u : 0u);
    };
    for (int j = 0; j < 2 && j < ntiles; ++j) {
      const int slot = take();
      qk(j, slot);
      tc_commit2_elect(&s_full[j]);
      tc_commit2_elect(&kv_empty[slot]);
    }
    for (int j = 0; j < ntiles; ++j) {
      const int buf = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      TR_TRACE_AT(0, j);
      const int vslot = take();
      TR_TRACE_AT(4, j);
      PAIR_WAIT(&p_full[buf * 2 + 0], ph);
      tc_fence_after();
      TR_TRACE_AT(1, j);
      TR_TRACE_GT(5, j);
      pv(buf, 0, vslot, j > 0);
      tc_commit2_elect(&pv_done[0]);
      PAIR_WAIT(&p_full[buf * 2 + 1], ph);
      tc_fence_after();
      TR_TRACE_AT(2, j);
      pv(buf, 1, vslot, j > 0);
      tc_commit2_elect(&pv_done[1]);
      tc_commit2_elect(&kv_empty[vslot]);
      if (j == ntiles - 1) tc_commit2_elect(o_done);
      if (j + 2 < ntiles) {
        const int kslot = take();
        qk(buf, kslot);
        tc_commit2_elect(&s_full[buf]);
        tc_commit2_elect(&kv_empty[kslot]);
      }
      TR_TRACE_AT(3, j);
    }
   }
  } else {
   setmaxnreg_inc<224>();
   {
    // ------------------------------------------------------------ softmax + epilogue
    const int g = (warp - 4) / 4;            // key group: columns [64g, 64g+64)
    const int quarter = warp % 4;            // TMEM lane quarter
    const int r = quarter * 32 + lane;       // row inside this CTA's 128 rows
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + 64 * g;       // + buf * 128
    const uint32_t tOg = tmem + lane_base + 256 + g * 128;
    const int64_t row_in_seg = my_row0 + r;
    const int64_t my_pos = Q.pos0 + row_in_seg;
    const int64_t tile_min_pos = Q.pos0 + my_row0;
    const float c = p.scale_log2;
    const float thresh = C::RESCALE_LOG2 / c;
    const uint64_t c2 = f2pack(c, c);
    const uint32_t pbar0 = mapa_u32(smem_u32(p_full), 0);   // leader's p_full[0]
    float m_used = -INFINITY;
    uint64_t lsum2[2] = {0ull, 0ull};
    KvWalk w = kv_begin(kv_tiles);
    for (int j = 0; j < ntiles; ++j, w.next(kv_tiles)) {
      const int buf = j & 1;
      const int64_t kpos = p.kv[w.g].pos0 + w.t * 128 + 64 * g;
      const int64_t left = p.kv[w.g].rows - w.t * 128 - 64 * g;
      const int valid = static_cast<int>(imax64(0, imin64(64, left)));
      TR_TRACE_AT(0, j);
      mbar_wait(&s_full[buf], (j >> 1) & 1);
      tc_fence_after();
      TR_TRACE_AT(1, j);
      uint32_t s[64];
      tmem_ld32_at<0>(tS + buf * 128, s);
      tmem_ld32_at<32>(tS + buf * 128 + 32, s);
      tc_wait_ld();
      const bool need_mask = valid < 64 || (p.causal && kpos + 63 > tile_min_pos);
      if (need_mask) {
        int64_t lim = valid;
        if (p.causal) lim = imin64(lim, my_pos - kpos + 1);
        const int limit = static_cast<int>(imax64(lim, 0));
        #pragma unroll
        for (int i = 0; i < 64; ++i) s[i] = (i < limit) ? s[i] : 0xFF800000u;  // -inf
      }
      float m4[4];
      #pragma unroll
      for (int a = 0; a < 4; ++a) {
        float m = __uint_as_float(s[16 * a]);
        #pragma unroll
        for (int i = 16 * a + 1; i < 16 * a + 15; i += 2)
          m = fmaxf(m, fmaxf(__uint_as_float(s[i]), __uint_as_float(s[i + 1])));
        m4[a] = fmaxf(m, __uint_as_float(s[16 * a + 15]));
      }
      const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      TR_TRACE_AT(2, j);
      const bool grow = mx > m_used + thresh;
      const bool scale_o = grow && m_used != -INFINITY;
      if (__any_sync(0xffffffffu, scale_o)) {
        // O_g may still be accumulating P_g(j-1).V_{j-1}: wait for it
        mbar_wait(&pv_done[g], (j - 1) & 1);
        tc_fence_after();
        const float f = scale_o ? ex2_approx((m_used - mx) * c) : 1.f;
        const uint64_t f2 = f2pack(f, f);
        lsum2[0] = fmul2(lsum2[0], f2);
        lsum2[1] = fmul2(lsum2[1], f2);
        #pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          uint32_t u[32];
          tmem_ld32(tOg + cc * 32, u);
          tc_wait_ld();
          #pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t v = fmul2(f2pack(__uint_as_float(u[i]), __uint_as_float(u[i + 1])), f2);
            u[i] = static_cast<uint32_t>(v);
            u[i + 1] = static_cast<uint32_t>(v >> 32);
          }
          tmem_st32(tOg + cc * 32, u);
        }
      }
      if (grow) m_used = mx;
      const float mc = (m_used == -INFINITY) ? 0.f : m_used * c;
      const uint64_t nmc2 = f2pack(-mc, -mc);
      uint32_t pk[32];
      if (need_mask) p_row64<C::POLY_MOD, false>(s, c2, nmc2, lsum2, pk);
      else p_row64<C::POLY_MOD, true>(s, c2, nmc2, lsum2, pk);
      tmem_st32(tS + buf * 128, pk);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      TR_TRACE_GT(5, j);
      if (lane == 0) mbar_arrive_cluster(pbar0 + 8u * (buf * 2 + g));
      TR_TRACE_AT(3, j);
    }
    float l;
    {
      float a0, a1, b0, b1;
      f2unpack(lsum2[0], a0, a1);
      f2unpack(lsum2[1], b0, b1);
      l = (a0 + a1) + (b0 + b1);
    }
    // ---------------------------------------------------------- epilogue
    if (ntiles > 0) {
      mbar_wait(o_done, 0);
      tc_fence_after();
    }
    float2* red = reinterpret_cast<float2*>(sQ);    // q tile is free once o_done fired
    red[g * 128 + r] = make_float2(m_used, l);
    named_barrier_sync(1, 256);
    const float2 other = red[(1 - g) * 128 + r];
    const float m = fmaxf(m_used, other.x);
    const float f_me = (m_used == -INFINITY) ? 0.f : ex2_approx((m_used - m) * c);
    const float f_ot = (other.x == -INFINITY) ? 0.f : ex2_approx((other.x - m) * c);
    const float L = l * f_me + other.y * f_ot;
    const float inv = (L > 0.f) ? 1.f / L : 0.f;
    const float fa = (g == 0 ? f_me : f_ot) * inv;
    const float fb = (g == 0 ? f_ot : f_me) * inv;
    const bool row_ok = row_in_seg < Q.rows;
    const int64_t grow_ = Q.row0 + row_in_seg;
    const int64_t oidx = (grow_ * p.heads + head) * D;
    const uint32_t tOA = tmem + lane_base + 256;
    const uint32_t tOB = tOA + 128;
    #pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int col = g * 64 + cc * 32;
      uint32_t ua[32], ub[32];
      if (ntiles > 0) {
        tmem_ld32(tOA + col, ua);
        tmem_ld32(tOB + col, ub);
        tc_wait_ld();
      } else {
        #pragma unroll
        for (int i = 0; i < 32; ++i) { ua[i] = 0u; ub[i] = 0u; }
      }
      float o[32];
      #pragma unroll
      for (int i = 0; i < 32; ++i)
        o[i] = __uint_as_float(ua[i]) * fa + __uint_as_float(ub[i]) * fb;
      if (!row_ok) continue;
      if (p.out_f32) {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + oidx + col);
        #pragma unroll
        for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
      } else {
        uint32_t pk[16];
        #pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(o[2 * i], o[2 * i + 1]);
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + oidx + col);
        #pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (row_ok && g == 0)
      p.lse[head * p.lse_stride + grow_] = (L > 0.f) ? (logf(L) + m * p.scale) : -INFINITY;
   }
  }
  tc_fence_before();
  if (p.done_flag) __threadfence_system();
  __syncthreads();
  cluster_sync();                            // the leader's MMAs read this CTA's smem/TMEM
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
  if (p.done_flag && threadIdx.x == 0) signal_done(p);
}

#endif  // TR_KERNEL_PAIR

// ------------------------------------------------------------------ host side
// one-CTA-per-item grid vs persistent CTAs: build default, overridable at run
// time with TR_ATTN_PERSISTENT=0/1
static bool use_persistent() {
#ifdef TR_PERSISTENT_DEFAULT
  bool v = TR_PERSISTENT_DEFAULT != 0;
#else
  bool v = false;
#endif
  if (const char* e = getenv("TR_ATTN_PERSISTENT")) v = e[0] == '1';
  return v;
}

// P in shared memory (attn_fwd_ps_kernel) vs in TMEM: build default,
// overridable at run time with TR_ATTN_PSMEM=0/1
static bool use_psmem() {
#ifdef TR_PSMEM_DEFAULT
  bool v = TR_PSMEM_DEFAULT != 0;
#else
  bool v = false;
#endif
  if (const char* e = getenv("TR_ATTN_PSMEM")) v = e[0] == '1';
  return v;
}

template <int D>
static int launch_persistent(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                             AttnPlan& plan, int64_t blocks, cudaStream_t s) {
  using C = AttnCfg<D>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_persistent_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(attn_fwd_persistent)");
    attr_done = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
    sms = 148;
  const int64_t grid = blocks < sms ? blocks : sms;
  attn_fwd_persistent_kernel<D><<<static_cast<unsigned>(grid), C::THREADS, C::SMEM, s>>>(tq, tk, tv, plan);
  return cuda_status(cudaGetLastError(), "attn_fwd_persistent launch");
}

int launch_attn_variant(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        AttnPlan& plan, int head_dim, int64_t blocks, cudaStream_t s) {
  if (head_dim == 128 && use_psmem()) {
    static bool ps_attr = false;
    if (!ps_attr) {
      cudaError_t e = cudaFuncSetAttribute(attn_fwd_ps_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, PsCfg::SMEM);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(attn_fwd_ps)");
      ps_attr = true;
    }
    attn_fwd_ps_kernel<<<static_cast<unsigned>(blocks), PsCfg::THREADS, PsCfg::SMEM, s>>>(tq, tk, tv, plan);
    return cuda_status(cudaGetLastError(), "attn_fwd_ps launch");
  }
  if (use_persistent()) {
    if (head_dim == 128) return launch_persistent<128>(tq, tk, tv, plan, blocks, s);
    if (head_dim == 64) return launch_persistent<64>(tq, tk, tv, plan, blocks, s);
  }
  return -1;
}

#ifdef TR_KERNEL_PAIR
int launch_attn_pair(const void* q, const void* k, const void* v, int64_t tq_total,
                       int64_t tk_total, AttnPlan& plan, cudaStream_t s) {
  using C = PairCfg;
  CUtensorMap tq, tk, tv;
  const int64_t row_elems = int64_t(plan.heads) * C::D;
  int rc;
  if ((rc = make_tmap(&tq, q, tq_total, row_elems, 128))) return rc;
  if ((rc = make_tmap(&tk, k, tk_total, row_elems, 64))) return rc;
  if ((rc = make_tmap(&tv, v, tk_total, row_elems, 128))) return rc;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_pair_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(attn_fwd_pair)");
    attr_done = true;
  }
  const int64_t pairs = plan.tile_prefix[plan.nq] * plan.heads;
  if (pairs == 0) return TR_OK;
  if (2 * pairs > 0x7FFFFFFF) return fail(TR_ERR_UNSUPPORTED, "grid too large");
  attn_fwd_pair_kernel<<<static_cast<unsigned>(2 * pairs), C::THREADS, C::SMEM, s>>>(tq, tk, tv, plan);
  return cuda_status(cudaGetLastError(), "attn_fwd_pair launch");
}
#endif  // TR_KERNEL_PAIR

#ifdef TR_TRACE
extern "C" int tr_debug_trace_variants(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_trace, bytes < sizeof(g_trace) ? bytes : sizeof(g_trace)) ==
                 cudaSuccess ? 0 : -4;
}
#endif

}  // namespace tr
