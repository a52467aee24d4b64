// Block attention forward for sm_100a: tcgen05 MMA with TMEM accumulators,
// TMA-staged Q/K/V tiles (128-byte swizzle), warp-specialised CTA.
//
// Computes, for every (q row i, head h) of the q segments against the union
// of the kv segments (ref _kernels_ref.py:34-54, _kernels.pyx:15-65):
//     lse(h,i) = log sum_j exp(s_ij),   out(i,h) = sum_j softmax(s)_ij v_j,
//     s_ij = q_i . k_j / sqrt(D),   causal: j visible iff pos(i) >= pos(j),
// rows without visible keys -> lse = -inf, out = 0.
//
// CTA = one head x 256 query rows (two 128-row tiles, "halves").
//   warp 0      TMA producer: Q once, then K_j / V_j into an NS-stage ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 4-7   softmax + epilogue for half 0   (TMEM lanes 0..127)
//   warps 8-11  softmax + epilogue for half 1
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [384,384+D);
// P_h (bf16, packed 2/col) overwrites S_h columns [0,64) once S_h is in
// registers, and is the A operand of the P.V MMA straight from TMEM.
// MMA issue order per kv tile j (keeps the tensor pipe busy while the two
// softmax groups alternate):  S0=Q0.Kj | O1+=P1.V(j-1) | S1=Q1.Kj | O0+=P0.Vj
// Online softmax keeps a stale running max unless it grows by > 8 (log2
// units): exact rescaling, done rarely, by the softmax warps themselves while
// the O accumulator is quiescent.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "attn_common.cuh"

namespace tr {

template <int D>
__global__ void __launch_bounds__(384, 1)
attn_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                      const __grid_constant__ CUtensorMap tmv, const __grid_constant__ AttnPlan p) {
  using C = AttnCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                      // 2 tiles
  uint8_t* sKV = smem + 2 * C::TILE;       // NS tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_TILES);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;                 // [NS]
  uint64_t* kv_empty = bars + 1 + C::NS;        // [NS]
  uint64_t* s_full = bars + 1 + 2 * C::NS;      // [2]
  uint64_t* p_full = bars + 3 + 2 * C::NS;      // [2 halves][NPC key chunks]
  uint64_t* o_done = p_full + 2 * C::NPC;       // [2]
  int64_t* kv_tiles = reinterpret_cast<int64_t*>(o_done + 2);  // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 6);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  int head;
  int qseg;
  int64_t qrow0;  // first row of this CTA inside its q segment
  cta_tile(p, blockIdx.x, head, qseg, qrow0);
  const tr_segment Q = p.q[qseg];
  const int64_t qmax_pos = Q.pos0 + imin64(qrow0 + 255, Q.rows - 1);

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::NS; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&s_full[h], 1);
      for (int kh = 0; kh < C::NPC; ++kh) mbar_init(&p_full[C::NPC * h + kh], 128);
      mbar_init(&o_done[h], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmq); tma_prefetch_desc(&tmk); tma_prefetch_desc(&tmv);
  }
  if (warp == 2 && lane < TR_MAX_SEGMENTS) {
    // kv tiles of every segment this q tile needs (causal: keys up to qmax_pos)
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
  // shared-memory loads are per-thread values to the compiler; broadcasting
  // them makes them provably warp-uniform (uniform-datapath MMA issue)
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int ntiles = __shfl_sync(
      0xffffffffu, static_cast<int>(kv_tiles[0] + kv_tiles[1] + kv_tiles[2] + kv_tiles[3]), 0);
  // resident: lets a programmatic dependent launch start on freed SMs (TR_LAUNCH_RELEASE_NEXT)
  if (p.release_next && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // Register rebalancing: each role's code sits inside the branch of its own
  // setmaxnreg so ptxas compiles it against that budget.
  if (warp < 4) {
   setmaxnreg_dec<56>();
   if (warp == 0 && ntiles > 0) {
    // ------------------------------------------------------------ producer
    // The whole warp walks the loop (warp-uniform state in uniform
    // registers); elect.sync inside each asm picks the issuing lane.
    const int32_t col0 = head * D;
    mbar_arrive_expect_tx_elect(q_full, 2 * C::TILE);
    for (int h = 0; h < 2; ++h)
      for (int b = 0; b < C::NB; ++b)
        tma_load_2d_elect(sQ + (h * C::NB + b) * C::BOX, &tmq, q_full, col0 + 64 * b,
                          static_cast<int32_t>(Q.row0 + qrow0 + 128 * h), kEvictFirst);
    KvWalk w = kv_begin(kv_tiles);
    int s = 0;
    uint32_t round = 0;
    for (int j = 0; j < ntiles; ++j, w.next(kv_tiles)) {
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
   } else if (warp == 1 && ntiles > 0) {
    // ------------------------------------------------------------ MMA issuer
    // one thread, elected once around the loop: plain tcgen05.mma / commit,
    // descriptors in uniform registers (as the pair kernel, attn_fwd_pair2.cu)
    if (elect_one_sync()) {
    const uint32_t q_addr = smem_u32(sQ);
    const uint32_t kv_addr = smem_u32(sKV);
    mbar_wait(q_full, 0);
    tc_fence_after();
    // Descriptors differ only in the start-address field (bits 0..13, in
    // 16-byte units), so each MMA adds an offset to one of three bases.
    const uint64_t dK = sdesc_sw128(kv_addr, 16, 1024);       // Q and K: K-major
    const uint64_t dQ = sdesc_sw128(q_addr, 16, 1024);
    const uint64_t dV = sdesc_sw128(kv_addr, C::BOX, 1024);   // V: MN-major
    auto qk = [&](int h, int stage) {
      const uint64_t a0 = dQ + static_cast<uint32_t>((h * C::TILE) >> 4);
      const uint64_t b0 = dK + static_cast<uint32_t>((stage * C::TILE) >> 4);
      #pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = ((kk / 4) * C::BOX + (kk % 4) * 32) >> 4;
        mma_ss(tmem + h * 128, desc_add(a0, off), desc_add(b0, off), C::IDESC_QK, kk > 0);
      }
    };
    // O_h += P_h[:, keys of chunk kh] . V[keys of chunk kh, :]
    constexpr int KPC = 8 / C::NPC;      // 16-key MMA steps per P chunk
    auto pv = [&](int h, int stage, int kh, bool acc) {
      const uint64_t b0 = dV + static_cast<uint32_t>((stage * C::TILE) >> 4);

      #pragma unroll
      for (int k4 = 0; k4 < KPC; ++k4) {
        const int kk = kh * KPC + k4;
#if defined(TR_EXP_NOSOFTMAX) && defined(TR_EXP_PSMEM)
        // experiment: A (P) from shared memory, SS mode
        const uint64_t a0 = dQ + static_cast<uint32_t>((h * C::TILE) >> 4);
        const uint32_t offa = ((kk / 4) * C::BOX + (kk % 4) * 32) >> 4;
        mma_ss(tmem + 256 + h * 128, desc_add(a0, offa), desc_add(b0, (kk * 2048) >> 4),
                     C::IDESC_PV, (acc || kk > 0) ? 1u : 0u);
#else
        mma_ts(tmem + 256 + h * 128, tmem + h * 128 + kk * 8, desc_add(b0, (kk * 2048) >> 4),
                     C::IDESC_PV, (acc || kk > 0) ? 1u : 0u);
#endif
      }
    };
    auto pv_both = [&](int h, int stage, uint32_t phase, bool acc) {
      #pragma unroll
      for (int kh = 0; kh < C::NPC; ++kh) {
        mbar_wait(&p_full[C::NPC * h + kh], phase);
        tc_fence_after();
        pv(h, stage, kh, acc || kh > 0);
      }
    };
    int prev_v_stage = 0;
    int sk = 0;
    uint32_t rk = 0;     // ring position / round of K_j (V_j follows it)
    for (int j = 0; j < ntiles; ++j) {
      const int sv = (sk + 1 == C::NS) ? 0 : sk + 1;
      const uint32_t rv = (sk + 1 == C::NS) ? rk + 1 : rk;
      mbar_wait(&kv_full[sk], rk & 1);
      tc_fence_after();
      TR_TRACE_AT(0, j);
      qk(0, sk);
      TR_TRACE_AT(1, j);
      tc_commit(&s_full[0]);
      if (j > 0) {
        pv_both(1, prev_v_stage, (j - 1) & 1, j - 1 > 0);
        tc_commit(&kv_empty[prev_v_stage]);
      }
      TR_TRACE_AT(2, j);
      qk(1, sk);
      tc_commit(&s_full[1]);
      tc_commit(&kv_empty[sk]);
      mbar_wait(&kv_full[sv], rv & 1);
      TR_TRACE_AT(3, j);
      pv_both(0, sv, j & 1, j > 0);
      TR_TRACE_AT(4, j);
      if (j == ntiles - 1) tc_commit(&o_done[0]);
      prev_v_stage = sv;
      sk = (sv + 1 == C::NS) ? 0 : sv + 1;
      rk = (sv + 1 == C::NS) ? rv + 1 : rv;
    }
    pv_both(1, prev_v_stage, (ntiles - 1) & 1, ntiles - 1 > 0);
    tc_commit(&kv_empty[prev_v_stage]);
    tc_commit(&o_done[1]);
    }
    __syncwarp();
   }
  } else {
   setmaxnreg_inc<224>();
   {
    // ------------------------------------------------------------ softmax + epilogue
    const int h = (warp - 4) / 4;         // which 128-row half
    const int quarter = warp % 4;         // TMEM lane quarter
    const int r = quarter * 32 + lane;    // row inside the half
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_base + h * 128;
    const uint32_t tO = tmem + lane_base + 256 + h * 128;
    const int64_t row_in_seg = qrow0 + 128 * h + r;
    const int64_t my_pos = Q.pos0 + row_in_seg;
    const int64_t half_min_pos = Q.pos0 + qrow0 + 128 * h;
    const float c = p.scale_log2;
    const float thresh = C::RESCALE_LOG2 / c;
    const uint64_t c2 = f2pack(c, c);
    float m_used = -INFINITY;
    uint64_t lsum2[2] = {0ull, 0ull};     // packed partial row sums
    KvWalk w = kv_begin(kv_tiles);
    for (int j = 0; j < ntiles; ++j, w.next(kv_tiles)) {
      const int64_t kpos = p.kv[w.g].pos0 + w.t * 128;
      const int valid = static_cast<int>(imin64(128, p.kv[w.g].rows - w.t * 128));
      TR_TRACE_AT(0, j);
      mbar_wait(&s_full[h], j & 1);
      TR_TRACE_AT(1, j);
      tc_fence_after();
#ifdef TR_EXP_NOSOFTMAX
      // experiment: measure the MMA/TMA pipeline alone (results are garbage)
#ifdef TR_EXP_PSMEM
      // ... with P written to shared memory (this half's Q tile stands in for
      // the P buffer: 256 B per row, 128B-swizzled K-major) for an SS-mode P.V
      {
        uint8_t* prow = sQ + h * C::TILE;
        #pragma unroll
        for (int c16 = 0; c16 < 16; ++c16) {
          const int box = c16 / 8, chunk = c16 % 8;
          uint4* dst = reinterpret_cast<uint4*>(prow + box * C::BOX + r * 128 + ((chunk ^ (r & 7)) * 16));
          *dst = make_uint4(r, c16, j, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
#endif
      tc_fence_before();
      for (int kh = 0; kh < C::NPC; ++kh) mbar_arrive(&p_full[C::NPC * h + kh]);
      continue;
#endif
      uint32_t s[128];
      // masking is decided per 128-row half (uniform across the warpgroup)
      const bool need_mask = valid < 128 || (p.causal && kpos + 127 > half_min_pos);
      tmem_ld32_at<0>(tS + 0, s);
      tmem_ld32_at<32>(tS + 32, s);
      tmem_ld32_at<64>(tS + 64, s);
      tmem_ld32_at<96>(tS + 96, s);
      tc_wait_ld();
      if (need_mask) {
        int64_t lim = valid;
        if (p.causal) lim = imin64(lim, my_pos - kpos + 1);
        const int limit = static_cast<int>(imax64(lim, 0));
        #pragma unroll
        for (int i = 0; i < 128; ++i) s[i] = (i < limit) ? s[i] : 0xFF800000u;  // -inf
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
      // tcgen05.ld/st are warp-collective: decide per warp, scale per row.
      if (__any_sync(0xffffffffu, scale_o)) {
        // O holds only completed P.V products (this tile's S commit implies
        // every earlier MMA finished); rescale it before publishing P_j.
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
      // P = exp2(s*c - m*c), bf16, written over S's first 64 columns in two
      // key halves so the P.V MMA can start on the first half early.  Masked
      // tiles keep every exp2 on MUFU (exact 0 for -inf); full tiles move one
      // pair in POLY_MOD to the FMA pipe.
      if (need_mask)
        emit_p<C::POLY_MOD, false, C::NPC>(s, tS, c2, nmc2, lsum2, &p_full[C::NPC * h]);
      else
        emit_p<C::POLY_MOD, true, C::NPC>(s, tS, c2, nmc2, lsum2, &p_full[C::NPC * h], j);
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
        // float32 rows straight into an (empty) accumulator: no bf16 round trip
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
  if (p.done_flag) __threadfence_system();   // out/lse rows may live on a peer GPU
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
  if (p.done_flag && threadIdx.x == 0) signal_done(p);
}

#ifdef TR_TRACE
extern "C" int tr_debug_trace(void* dst, size_t bytes) {
  return cudaMemcpyFromSymbol(dst, g_trace, bytes < sizeof(g_trace) ? bytes : sizeof(g_trace)) ==
                 cudaSuccess ? 0 : -4;
}
#endif

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

int make_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t row_elems,
              uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(TR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_elems), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_elems * 2)};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TR_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return TR_OK;
}

bool sm100_supports(int head_dim, int heads, const void* q, const void* k, const void* v,
                    const void* out) {
  if (head_dim != 64 && head_dim != 128) return false;
  const int64_t row_bytes = int64_t(heads) * head_dim * 2;
  if (row_bytes % 16) return false;
  for (const void* ptr : {q, k, v, out})
    if (reinterpret_cast<uintptr_t>(ptr) % 16) return false;
  return true;
}

template <int D>
static int launch_d(const void* q, const void* k, const void* v, int64_t tq_total, int64_t tk_total,
                    AttnPlan& plan, cudaStream_t s) {
  using C = AttnCfg<D>;
  CUtensorMap tq, tk, tv;
  const int64_t row_elems = int64_t(plan.heads) * D;
  int rc;
  if ((rc = make_tmap(&tq, q, tq_total, row_elems))) return rc;
  if ((rc = make_tmap(&tk, k, tk_total, row_elems))) return rc;
  if ((rc = make_tmap(&tv, v, tk_total, row_elems))) return rc;
  int rc2;
  if ((rc2 = set_smem_attr_once(reinterpret_cast<const void*>(attn_fwd_sm100_kernel<D>), C::SMEM,
                                "cudaFuncSetAttribute(attn_fwd_sm100)")))
    return rc2;
  const int64_t blocks = plan.tile_prefix[plan.nq] * plan.heads;
  if (blocks == 0) return TR_OK;
  if (blocks > 0x7FFFFFFF) return fail(TR_ERR_UNSUPPORTED, "grid too large");
#ifdef TR_EXPERIMENTS
  // experiments build only: measured-and-rejected alternatives (TR_ATTN_PSMEM /
  // TR_ATTN_PERSISTENT, attn_fwd_variants.cu); the product library has no
  // run-time kernel switch
  const int vrc = launch_attn_variant(tq, tk, tv, plan, D, blocks, s);
  if (vrc != -1) return vrc;
#endif
  return cuda_status(launch_kernel(attn_fwd_sm100_kernel<D>, dim3(static_cast<unsigned>(blocks)),
                                   dim3(C::THREADS), C::SMEM, s, plan.overlap_prev != 0, tq, tk,
                                   tv, plan),
                     "attn_fwd_sm100 launch");
}


#ifdef TR_EXPERIMENTS
// experiments build: D=128 on the single-CTA kernel with TR_ATTN_PAIR2=0 or one
// of the single-CTA variants (A/B and the pair-vs-single parity test only)
static bool use_pair2() {
  static int v = -1;
  if (v < 0) {
    v = 1;
    if (const char* e = getenv("TR_ATTN_PAIR2")) v = e[0] == '1';
    for (const char* name : {"TR_ATTN_PSMEM", "TR_ATTN_PERSISTENT"})
      if (const char* e = getenv(name))
        if (e[0] == '1') v = 0;
  }
  return v == 1;
}
#else
static constexpr bool use_pair2() { return true; }
#endif

int launch_attn_sm100(const void* q, const void* k, const void* v, int64_t tq_total,
                      int64_t tk_total, int head_dim, AttnPlan& plan, cudaStream_t s) {
#ifdef TR_KERNEL_PAIR
  if (head_dim == 128) return launch_attn_pair(q, k, v, tq_total, tk_total, plan, s);
#else
  if (head_dim == 128 && use_pair2()) return launch_attn_pair2(q, k, v, tq_total, tk_total, plan, s);
  if (head_dim == 128) return launch_d<128>(q, k, v, tq_total, tk_total, plan, s);
#endif
  if (head_dim == 64) return launch_d<64>(q, k, v, tq_total, tk_total, plan, s);
  return fail(TR_ERR_UNSUPPORTED, "sm100 attention kernel supports head_dim 64 or 128");
}

}  // namespace tr
