// consensus_tma.cuh -- persistent, TMA-pipelined consensus pass (K2) for
// uniform tilings with 64- or 128-wide blocks.  Included by dope_lattice.cu
// inside namespace dope (uses Lat2, reduce_blocks, finalize_apply, other_buffer).
//
// Same arithmetic as k_consensus_vec (solve_global + clamp admm.py:194-238,
// update_multipliers admm.py:241-248, block residuals admm.py:251-257, energy
// of the previous iterate energy.py:187-194), organised for HBM:
//   * persistent grid (a few CTAs per SM); each CTA walks its blocks as tiles
//     of TH x TW pixels (64x64, or 32 rows of a 128-wide block);
//   * per tile, one thread issues 2D TMA loads (cp.async.bulk.tensor) of the
//     int16 multipliers, the uint8 iterate y2 (+ the row below), the y2
//     column right of the tile and the label tile with a 1-row / 16-byte halo
//     into a STAGES-deep shared-memory ring, completion tracked by mbarriers;
//     u is not streamed (the unary energy is kept incrementally);
//   * results go straight from registers to HBM (8-byte multiplier quads,
//     4-byte iterate quads);
//   * per-block partials are accumulated with one atomic per warp (the next
//     K1 clears them); each CTA then folds its own blocks into pass-wide
//     aggregates, so the last CTA only adds up one residual sum per CTA.

struct TmaMaps {
    CUtensorMap a[2], y[3], yr[3], yhat;
};

// Stage layout of one TH x TW tile: multipliers (int16), previous iterate y2
// (uint8, +1 row below), the 16-byte column right of the tile (its first byte is
// the right-halo y2), labels with a 1-row / 16-byte halo.  u is not streamed:
// the unary energy is kept incrementally (u gathered only where y changes).
template <int TW, int NT_ = 512, int STAGES_ = 3>
struct TmaCfg {
    static constexpr int TH = 4096 / TW;                 // tile rows (64 or 32)
    static constexpr int NT = NT_;
    static constexpr int QPT = TH * TW / 4 / NT;         // quads per thread
    static constexpr int YHW = TW + 32;                  // label box width (bytes)
    static constexpr int B_A = TW * TH * 2;
    static constexpr int B_Y = TW * (TH + 1);
    static constexpr int B_YR = 16 * TH;
    static constexpr int B_H = YHW * (TH + 2);
    static constexpr int O_A = 0;
    static constexpr int O_Y = (O_A + B_A + 127) / 128 * 128;
    static constexpr int O_YR = (O_Y + B_Y + 127) / 128 * 128;
    static constexpr int O_H = (O_YR + B_YR + 127) / 128 * 128;
    static constexpr int STAGE = (O_H + B_H + 127) / 128 * 128;
    static constexpr int TX = B_A + B_Y + B_YR + B_H;
    static constexpr int STAGES = STAGES_;
    static constexpr int SMEM = STAGES * STAGE + 128;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x,
                                            int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

template <int TW>
__device__ __forceinline__ void tma_issue_tile(const Lat2 &L, const TmaMaps &M, uint8_t *stage,
                                               uint64_t *bar, int by, int bx, int tile, int cur, int p) {
    using C = TmaCfg<TW>;   // box geometry does not depend on NT / STAGES
    const int x0 = bx * TW;                       // uniform tiling: lo = index * width
    const int y0 = by * L.ay.base + tile * C::TH;
    mbar_expect_tx(bar, C::TX);
    tma_load_2d(stage + C::O_A, &M.a[p], bar, x0, y0);
    // y / labels maps start at the ghost row above the shard: +1 row
    tma_load_2d(stage + C::O_Y, &M.y[cur], bar, x0, y0 + 1);
    tma_load_2d(stage + C::O_YR, &M.yr[cur], bar, x0 + TW, y0 + 1);
    tma_load_2d(stage + C::O_H, &M.yhat, bar, x0 - 16, y0);
}

// 4 bytes (each 0 or 1) -> 4 bits
__device__ __forceinline__ uint32_t bits_b01(uint32_t w) { return ((w * 0x01020408u) >> 24) & 0xFu; }
// 4 bits -> 4 bytes (each 0 or 1)
__device__ __forceinline__ uint32_t bytes_b01(uint32_t b) { return (b * 0x00204081u) & 0x01010101u; }

// One quad (4 consecutive pixels of a row) of the consensus update.
//   h4  : labels (bytes 0/1)         a2  : multipliers (int16 x 4)
//   cnt : per-pixel count of cross-block neighbours (bytes)
//   nb  : per-pixel sum of their labels (bytes)
// y = clamp(h + a - q * sx) with sx = cnt*h - nb (the solve_global stencil,
// admm.py:194-238); sx enters biased by 4 so the bytewise subtraction never
// borrows.  Returns the new y as bits; writes the new multipliers.
__device__ __forceinline__ uint32_t quad_update(uint32_t h4, uint2 a2, uint32_t cnt, uint32_t nb, int q,
                                                int q4, uint2 &an, uint32_t &clp) {
    const uint32_t sb = ((cnt & (h4 * 0xFFu)) | 0x04040404u) - nb;   // bytes: sx + 4
    const int a0 = (int)__byte_perm(a2.x, 0, 0x9910), a1 = (int)a2.x >> 16;
    const int a3_ = (int)a2.y >> 16, a2_ = (int)__byte_perm(a2.y, 0, 0x9910);
    const int h0 = __byte_perm(h4, 0, 0x4440), h1 = __byte_perm(h4, 0, 0x4441);
    const int h2 = __byte_perm(h4, 0, 0x4442), h3 = __byte_perm(h4, 0, 0x4443);
    const int p0 = a0 + h0 + q4 - q * (int)__byte_perm(sb, 0, 0x4440);
    const int p1 = a1 + h1 + q4 - q * (int)__byte_perm(sb, 0, 0x4441);
    const int p2 = a2_ + h2 + q4 - q * (int)__byte_perm(sb, 0, 0x4442);
    const int p3 = a3_ + h3 + q4 - q * (int)__byte_perm(sb, 0, 0x4443);
    clp |= (uint32_t)(p0 | p1) | (uint32_t)(p2 | p3);   // all in {0,1} <=> OR <= 1
    const int y0 = p0 > 0, y1 = p1 > 0, y2 = p2 > 0, y3 = p3 > 0;
    an.x = __byte_perm((uint32_t)(a0 + h0 - y0), (uint32_t)(a1 + h1 - y1), 0x5410);
    an.y = __byte_perm((uint32_t)(a2_ + h2 - y2), (uint32_t)(a3_ + h3 - y3), 0x5410);
    return (uint32_t)(y0 | (y1 << 1) | (y2 << 2) | (y3 << 3));
}

template <int TW, int NT_, int STAGES_>
__global__ void __launch_bounds__(NT_, (NT_ <= 128 ? 4 : (NT_ <= 256 ? 2 : 1))) k_consensus_tma(Lat2 L, const __grid_constant__ TmaMaps M,
                                                          uint32_t kx_magic) {
    using C = TmaCfg<TW, NT_, STAGES_>;
    constexpr int TH = C::TH, NT = C::NT, QPT = C::QPT, QR = TW / 4, LQ = (TW == 64) ? 4 : 5;
    extern __shared__ __align__(128) uint8_t smem_t[];
    // keep the shared address space visible to the compiler (LDS, not generic LD)
    uint8_t *base = smem_t + ((128u - (smem_u32(smem_t) & 127u)) & 127u);
    __shared__ __align__(8) uint64_t full[C::STAGES];
    __shared__ int last;
    // per-block accumulators, double-buffered by block parity: warps add into
    // acc[kb & 1] before the block's last barrier, thread 0 drains it after
    __shared__ unsigned long long accU[2];
    __shared__ unsigned int accE[2], accS[2], accF[2];

    dope_run_state *st = L.st;
    if (st->stop) return;
    const int tid = threadIdx.x, lane = tid & 31;
    if (L.timeline && tid == 0) {   // diagnostics: CTA start (slot 6 of entry blockIdx)
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        L.timeline[8 * blockIdx.x + 6] = (int64_t)t;
    }
    const int cur = st->ycur, best = st->ybest, out = other_buffer(cur, best);
    const int p = st->parity;
    ystore_t *__restrict__ y_out = L.y2[out];
    astore_t *__restrict__ a_out = p ? L.a0 : L.a1;
    const bool want_e = st->iteration >= 1;
    const int32_t W = L.W, H = L.ay.dim, q = L.q, BH = L.ay.base, KX = L.ax.k;
    const int q4 = 4 * q;
    const int tpb = BH / TH;                          // tiles per block
    const int G0 = gridDim.x;
    const int nblk = (L.K - (int)blockIdx.x + G0 - 1) / G0;
    const int ntiles = nblk * tpb;
    auto coords = [&](int kb, int &by, int &bx) {
        const int k = blockIdx.x + kb * G0;
        by = (int)__umulhi((uint32_t)k, kx_magic);
        bx = k - by * KX;
    };

    int ikb = 0, itile = 0;
    // thread 0: this CTA's pass aggregates (blocks in a fixed order)
    int64_t cE = 0, cU = 0, cM = -1;
    double cR = 0.0;
    int cF = 0;
    if (tid < 2) {
        accU[tid] = 0;
        accE[tid] = 0;
        accS[tid] = 0;
        accF[tid] = 0;
    }
    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < C::STAGES && i < ntiles; ++i) {
            int by, bx;
            coords(ikb, by, bx);
            tma_issue_tile<TW>(L, M, base + i * C::STAGE, &full[i], by, bx, itile, cur, p);
            if (++itile == tpb) { itile = 0; ++ikb; }
        }
    }
    __syncthreads();

    int rr_[QPT], c0_[QPT];
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int t = tid + j * NT;
        rr_[j] = t >> LQ;
        c0_[j] = (t & (QR - 1)) << 2;
    }

    int s = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < nblk; ++kb) {
        int by, bx;
        coords(kb, by, bx);
        const int k = by * KX + bx;
        const int lo_r = by * BH, lo_c = bx * TW;
        const bool has_up = lo_r > 0 || L.gup, has_dn = lo_r + BH < H || L.gdn, has_lf = lo_c > 0,
                   has_rt = lo_c + TW < W;
        const bool last_row_pairs = lo_r + BH < H || L.gdn;   // pairs below the block's last row
        int64_t du = 0;
        int ss = 0, quad_acc = 0;
        uint32_t fl = 0, clp = 0;   // fl: bit1 self, bit2 left, bit3 right, bit4 up, bit5 down
        for (int tile = 0; tile < tpb; ++tile) {
            const uint8_t *sb = base + s * C::STAGE;
            const astore_t *sa = reinterpret_cast<const astore_t *>(sb + C::O_A);
            const uint8_t *sy = sb + C::O_Y;
            const uint8_t *syr = sb + C::O_YR;
            const uint8_t *sh = sb + C::O_H + C::YHW + 16;      // label of tile pixel (0,0)
            const int r0 = tile * TH;
            const int64_t gt = (int64_t)(lo_r + r0) * W + lo_c;   // global index of tile (0,0)
            mbar_wait(&full[s], phase);
#pragma unroll
            for (int j = 0; j < QPT; ++j) {
                const int rr = rr_[j], c0 = c0_[j];
                const int r = r0 + rr;                             // row within block
                const uint2 av = *reinterpret_cast<const uint2 *>(sa + rr * TW + c0);
                const uint32_t yo = *reinterpret_cast<const uint32_t *>(sy + rr * TW + c0);
                const uint8_t *hrow = sh + rr * C::YHW + c0;
                const uint32_t h4 = *reinterpret_cast<const uint32_t *>(hrow);
                const bool cr = c0 + 4 == TW;
                if (want_e) {
                    // E(y_{t-1}) pair terms: bytes are 0/2, so each differing
                    // pair is exactly one set bit of the XOR
                    const uint32_t nxt = __shfl_down_sync(FULLMASK, yo, 1);
                    uint32_t rw = nxt;
                    if (cr) rw = has_rt ? (uint32_t)syr[rr * 16] : (yo >> 24);
                    const uint32_t yb = (r + 1 < BH || last_row_pairs)
                                            ? *reinterpret_cast<const uint32_t *>(sy + (rr + 1) * TW + c0)
                                            : yo;
                    quad_acc += __popc(yo ^ __funnelshift_r(yo, rw, 8)) + __popc(yo ^ yb);
                }
                // cross-block neighbours of this quad
                const bool lft = (c0 == 0) && has_lf, rgt = cr && has_rt;
                const bool top = (r == 0) && has_up, bot = (r == BH - 1) && has_dn;
                uint32_t cnt = 0, nb = 0;
                if (top) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(hrow - C::YHW); }
                if (bot) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(hrow + C::YHW); }
                if (lft) { cnt += 1u; nb += hrow[-1]; }
                if (rgt) { cnt += 1u << 24; nb += (uint32_t)hrow[4] << 24; }
                uint2 an;
                const uint32_t yn = quad_update(h4, av, cnt, nb, q, q4, an, clp);
                const uint32_t hb = bits_b01(h4);
                ss += __popc(hb ^ yn);
                const uint32_t yw = bytes_b01(yn) << 1;            // y2 bytes 0/2
                const uint32_t chg = yw ^ yo;
                fl |= (chg | (hb ^ yn)) ? 2u : 0u;
                const int64_t G = gt + (int64_t)rr * W + c0;
                __stcs(reinterpret_cast<uint2 *>(a_out + G), an);
                __stcg(reinterpret_cast<unsigned int *>(y_out + G), yw);
                if (chg) {
                    // running unary term u * (y2_new - y2_old) where y moved
                    const int4 uv = __ldg(reinterpret_cast<const int4 *>(L.u + G));
                    du += (int64_t)uv.x * ((int)(yw & 0xFFu) - (int)(yo & 0xFFu)) +
                          (int64_t)uv.y * ((int)((yw >> 8) & 0xFFu) - (int)((yo >> 8) & 0xFFu)) +
                          (int64_t)uv.z * ((int)((yw >> 16) & 0xFFu) - (int)((yo >> 16) & 0xFFu)) +
                          (int64_t)uv.w * ((int)(yw >> 24) - (int)(yo >> 24));
                    const uint32_t em = (lft ? 4u : 0u) | (rgt ? 8u : 0u) | (top ? 16u : 0u) | (bot ? 32u : 0u);
                    const uint32_t mk = 0x30u | ((chg & 0xFFu) ? 4u : 0u) | ((chg >> 24) ? 8u : 0u);
                    fl |= em & mk;
                }
            }
            const int ab = kb & 1;
            if (tile == tpb - 1) {
                // block done in this warp: one shared atomic per quantity
                const unsigned e = __reduce_add_sync(FULLMASK, (unsigned)quad_acc);
                const unsigned sq = __reduce_add_sync(FULLMASK, (unsigned)ss);
                const unsigned f = __reduce_or_sync(FULLMASK, fl | (clp > 1u ? 1u : 0u));
                int64_t u2 = 0;
                if (__any_sync(FULLMASK, du != 0)) u2 = warp_sum(du);
                if (lane == 0) {
                    if (e) atomicAdd(&accE[ab], e);
                    if (sq) atomicAdd(&accS[ab], sq);
                    if (f) atomicOr(&accF[ab], f);
                    if (u2) atomicAdd(&accU[ab], (unsigned long long)u2);
                }
            }
            // every warp is done with stage s: refill it with the tile STAGES ahead
            __syncthreads();
            if (tid == 0) {
                if (ikb < nblk) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    int by2, bx2;
                    coords(ikb, by2, bx2);
                    tma_issue_tile<TW>(L, M, base + s * C::STAGE, &full[s], by2, bx2, itile, cur, p);
                    if (++itile == tpb) { itile = 0; ++ikb; }
                }
                if (tile == tpb - 1) {
                    // drain block k: per-block partials (diagnostics / step API
                    // parity), dirty marks, and this CTA's running aggregates
                    const int64_t e = (int64_t)L.lamw * accE[ab];
                    const int64_t u2 = (int64_t)accU[ab];
                    const int64_t sq = accS[ab];
                    const unsigned f = accF[ab];
                    accE[ab] = 0;
                    accS[ab] = 0;
                    accF[ab] = 0;
                    accU[ab] = 0;
                    L.pe[k] = e;
                    L.pu[k] = u2;
                    L.pr[k] = sq;
                    L.pf[k] = (int)(f & 1u);
                    cE += e;
                    cU += u2;
                    cM = sq > cM ? sq : cM;
                    const double r = sqrt((double)sq);
                    cR += r * r;
                    cF |= (int)(f & 1u);
                    if (f & 2u) L.dirty[k] = 1u;
                    if (f & 4u) L.dirty[k - 1] = 1u;
                    if (f & 8u) L.dirty[k + 1] = 1u;
                    if ((f & 16u) && k - KX >= 0) L.dirty[k - KX] = 1u;
                    if ((f & 32u) && k + KX < L.K) L.dirty[k + KX] = 1u;
                }
            }
            if (++s == C::STAGES) { s = 0; phase ^= 1u; }
        }
    }
    // fold this CTA's aggregates into the pass-wide ones (exact integer
    // atomics; the float residual sum per CTA, for the last CTA to add up by
    // CTA index -- deterministic)
    // this CTA's blocks are complete: fold their partials into the pass-wide
    // aggregates (exact integer atomics; the float residual sum per CTA, in a
    // fixed order, for the last CTA to add up by CTA index)
    if (tid == 0) {
        atomicAdd(reinterpret_cast<unsigned long long *>(&L.pc[0]), (unsigned long long)cE);
        atomicAdd(reinterpret_cast<unsigned long long *>(&L.pc[1]), (unsigned long long)cU);
        atomicMax(reinterpret_cast<unsigned long long *>(&L.pc[2]), (unsigned long long)(cM + 1));
        if (cF) atomicOr(reinterpret_cast<unsigned long long *>(&L.pc[3]), 1ull);
        L.pc[8 + blockIdx.x] = __double_as_longlong(cR);
        if (L.timeline) {   // diagnostics: CTA end (slot 7)
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            L.timeline[8 * blockIdx.x + 7] = (int64_t)t;
        }
        __threadfence();
        const int prev = atomicAdd(&st->done_ctas, 1);
        last = (prev == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        dope_run_state s0;
        int64_t E2 = 0, U2 = 0, M2 = 0, F2 = 0;
        if (tid == 0) {   // in flight together with the residual loads
            s0 = *st;
            E2 = __ldcg(&L.pc[0]);
            U2 = __ldcg(&L.pc[1]);
            M2 = __ldcg(&L.pc[2]) - 1;
            F2 = __ldcg(&L.pc[3]);
        }
        // residual sum over CTAs in index order (deterministic)
        __shared__ double sR[NT_ / 32];
        double R = 0.0;
        for (int i = tid; i < (int)gridDim.x; i += NT) R += __longlong_as_double(__ldcg(&L.pc[8 + i]));
        for (int o = 16; o > 0; o >>= 1) R += __shfl_xor_sync(FULLMASK, R, o);
        if (lane == 0) sR[tid >> 5] = R;
        __syncthreads();
        if (tid == 0) {
            double R2 = 0.0;
            for (int w = 0; w < NT / 32; ++w) R2 += sR[w];
            L.pc[0] = 0;
            L.pc[1] = 0;
            L.pc[2] = 0;
            L.pc[3] = 0;
            finalize_apply(L, s0, E2, U2, R2, M2, (int)F2, cur, best, out);
            st->done_ctas = 0;
            if (L.timeline && (int)gridDim.x < L.K) {   // diagnostics: finalize end
                uint64_t t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                L.timeline[8 * gridDim.x + 7] = (int64_t)t;
            }
        }
    }
}
