// consensus_tma.cuh -- persistent, TMA-pipelined consensus pass (K2) for
// uniform tilings with 64- or 128-wide blocks.  Included by dope_lattice.cu
// inside namespace dope (uses Lat2, finalize_cta, other_buffer, warp_sum).
//
// Same arithmetic as k_consensus_vec (solve_global + clamp admm.py:194-238,
// update_multipliers admm.py:241-248, block residuals admm.py:251-257, energy
// of the previous iterate energy.py:187-194), organised for HBM:
//   * grid = one CTA per SM; each CTA walks its blocks as tiles of TH x TW
//     pixels (64x64, or 32 rows of a 128-wide block);
//   * per tile, one thread issues 2D TMA loads (cp.async.bulk.tensor) of u,
//     a, y (+ the row below), the y column right of the tile and the label
//     tile with a 1-row / 16-byte halo into a 3-stage shared-memory ring,
//     completion tracked by mbarriers -- two tiles are always in flight while
//     the CTA computes the third;
//   * results go straight from registers to HBM (16-byte streaming stores);
//   * per-block partials are accumulated with one atomic per warp; the last
//     CTA runs finalize_cta, which also clears them for the next iteration.

struct TmaMaps {
    CUtensorMap u, a[2], y[3], yr[3], yhat;
};

template <int TW, int NT_ = 512, int STAGES_ = 3>
struct TmaCfg {
    static constexpr int TH = 4096 / TW;                 // tile rows (64 or 32)
    static constexpr int NT = NT_;
    static constexpr int QPT = TH * TW / 4 / NT;         // quads per thread (2)
    static constexpr int YHW = TW + 32;                  // label box width (bytes)
    static constexpr int B_U = TW * TH * 4;
    static constexpr int B_A = TW * TH * 4;
    static constexpr int B_Y = TW * (TH + 1) * 4;
    static constexpr int B_YR = 4 * TH * 4;
    static constexpr int B_H = YHW * (TH + 2);
    static constexpr int O_U = 0;
    static constexpr int O_A = O_U + B_U;
    static constexpr int O_Y = O_A + B_A;
    static constexpr int O_YR = (O_Y + B_Y + 127) / 128 * 128;
    static constexpr int O_H = (O_YR + B_YR + 127) / 128 * 128;
    static constexpr int STAGE = (O_H + B_H + 127) / 128 * 128;
    static constexpr int TX = B_U + B_A + B_Y + B_YR + B_H;
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
    tma_load_2d(stage + C::O_U, &M.u, bar, x0, y0);
    tma_load_2d(stage + C::O_A, &M.a[p], bar, x0, y0);
    // y / labels maps start at the ghost row above the shard: +1 row
    tma_load_2d(stage + C::O_Y, &M.y[cur], bar, x0, y0 + 1);
    tma_load_2d(stage + C::O_YR, &M.yr[cur], bar, x0 + TW, y0 + 1);
    tma_load_2d(stage + C::O_H, &M.yhat, bar, x0 - 16, y0);
}

// packed old-iterate bits of a quad: y2 in {0,2} -> bit i = y_i
__device__ __forceinline__ uint32_t pack_y2(const int4 v) {
    return (uint32_t)((v.x | (v.y << 1) | (v.z << 2) | (v.w << 3)) >> 1);
}

template <int TW, int NT_, int STAGES_>
__global__ void __launch_bounds__(NT_, 1) k_consensus_tma(Lat2 L, const __grid_constant__ TmaMaps M,
                                                          uint32_t kx_magic) {
    using C = TmaCfg<TW, NT_, STAGES_>;
    constexpr int TH = C::TH, NT = C::NT, QPT = C::QPT, QR = TW / 4, LQ = (TW == 64) ? 4 : 5;
    extern __shared__ __align__(128) uint8_t smem_t[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_t) + 127) & ~(uintptr_t)127);
    __shared__ __align__(8) uint64_t full[C::STAGES];
    __shared__ int last;

    dope_run_state *st = L.st;
    if (st->stop) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const int cur = st->ycur, best = st->ybest, out = other_buffer(cur, best);
    const int p = st->parity;
    int32_t *__restrict__ y_out = L.y2[out];
    int32_t *__restrict__ a_out = p ? L.a0 : L.a1;
    const bool want_e = st->iteration >= 1;
    const int32_t W = L.W, H = L.ay.dim, q = L.q, BH = L.ay.base, KX = L.ax.k;
    const int tpb = BH / TH;                          // tiles per block
    const int G0 = gridDim.x;
    const int nblk = (L.K - (int)blockIdx.x + G0 - 1) / G0;
    const int ntiles = nblk * tpb;
    // block coordinates of this CTA's kb-th block (division-free: magic = ceil(2^32 / KX))
    auto coords = [&](int kb, int &by, int &bx) {
        const int k = blockIdx.x + kb * G0;
        by = (int)__umulhi((uint32_t)k, kx_magic);
        bx = k - by * KX;
    };

    // issue cursor (thread 0 only)
    int ikb = 0, itile = 0;
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

    // per-thread quad positions inside a tile (fixed for the whole launch)
    int off_[QPT], goff_[QPT], rr_[QPT];
    bool cl_[QPT], cr_[QPT];
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int t = tid + j * NT;
        const int rr = t >> LQ, c0 = (t & (QR - 1)) << 2;
        rr_[j] = rr;
        off_[j] = rr * TW + c0;           // smem offset in the tile
        goff_[j] = rr * W + c0;           // global offset from the tile origin
        cl_[j] = c0 == 0;
        cr_[j] = c0 + 4 == TW;
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
        int64_t e_acc = 0;
        int ss = 0, quad_acc = 0;
        bool clamped = false, chg_self = false, chgL = false, chgR = false, chgU = false, chgD = false;
        for (int tile = 0; tile < tpb; ++tile) {
            uint8_t *sb = base + s * C::STAGE;
            const int32_t *su = reinterpret_cast<const int32_t *>(sb + C::O_U);
            const int32_t *sa = reinterpret_cast<const int32_t *>(sb + C::O_A);
            const int32_t *sy = reinterpret_cast<const int32_t *>(sb + C::O_Y);
            const int32_t *syr = reinterpret_cast<const int32_t *>(sb + C::O_YR);
            const uint8_t *sh = sb + C::O_H + C::YHW + 16;      // label of tile pixel (0,0)
            const int r0 = tile * TH;
            int32_t *a_t = a_out + (int64_t)(lo_r + r0) * W + lo_c;
            int32_t *y_t = y_out + (int64_t)(lo_r + r0) * W + lo_c;
            mbar_wait(&full[s], phase);
#pragma unroll
            for (int j = 0; j < QPT; ++j) {
                const int rr = rr_[j], off = off_[j];
                const int r = r0 + rr;                             // row within block
                const int4 av = *reinterpret_cast<const int4 *>(sa + off);
                const int4 yo = *reinterpret_cast<const int4 *>(sy + off);
                const int4 uu = *reinterpret_cast<const int4 *>(su + off);
                const uint8_t *hrow = sh + rr * C::YHW + (off - rr * TW);
                const uint32_t yh4 = *reinterpret_cast<const uint32_t *>(hrow);
                // old iterate (y2 in {0,2} from iteration 2 on) as 4 bits
                const uint32_t ob = pack_y2(yo);
                const uint32_t nxt = __shfl_down_sync(FULLMASK, ob, 1);
                if (want_e) {
                    const int4 yb = *reinterpret_cast<const int4 *>(sy + off + TW);
                    uint32_t rb = nxt;
                    if (cr_[j]) rb = has_rt ? (uint32_t)(syr[rr * 4] >> 1) : (ob >> 3);
                    const uint32_t hz = (ob ^ (ob >> 1)) & 0x7u;                 // pairs inside the quad
                    const uint32_t vt = (lo_r + r + 1 < H || L.gdn) ? (ob ^ pack_y2(yb)) : 0u;
                    quad_acc += __popc(hz | (((ob >> 3) ^ rb) & 1u) << 3) + __popc(vt);
                    e_acc += uu.x * (yo.x >> 1) + uu.y * (yo.y >> 1) + uu.z * (yo.z >> 1) +
                             uu.w * (yo.w >> 1);
                }
                const int h0 = yh4 & 0xFF, h1 = (yh4 >> 8) & 0xFF, h2 = (yh4 >> 16) & 0xFF, h3 = yh4 >> 24;
                // cross-block sums (non-zero only on the block border)
                const bool lft = cl_[j] && has_lf, rgt = cr_[j] && has_rt;
                int sx0 = lft ? h0 - (int)hrow[-1] : 0;
                int sx3 = rgt ? h3 - (int)hrow[4] : 0;
                int sx1 = 0, sx2 = 0;
                const bool top = (r == 0) && has_up, bot = (r == BH - 1) && has_dn;
                if (top | bot) {
                    const uint32_t o4 = *reinterpret_cast<const uint32_t *>(hrow + (top ? -C::YHW : C::YHW));
                    sx0 += h0 - (int)(o4 & 0xFF);
                    sx1 += h1 - (int)((o4 >> 8) & 0xFF);
                    sx2 += h2 - (int)((o4 >> 16) & 0xFF);
                    sx3 += h3 - (int)(o4 >> 24);
                    if (top && bot) {   // single-row blocks: both neighbours
                        const uint32_t d4 = *reinterpret_cast<const uint32_t *>(hrow + C::YHW);
                        sx0 += h0 - (int)(d4 & 0xFF);
                        sx1 += h1 - (int)((d4 >> 8) & 0xFF);
                        sx2 += h2 - (int)((d4 >> 16) & 0xFF);
                        sx3 += h3 - (int)(d4 >> 24);
                    }
                }
                const int p0 = h0 + av.x - q * sx0, p1 = h1 + av.y - q * sx1;
                const int p2 = h2 + av.z - q * sx2, p3 = h3 + av.w - q * sx3;
                clamped |= (unsigned)(p0 | p1 | p2 | p3) > 1u;
                const int y0 = min(max(p0, 0), 1), y1 = min(max(p1, 0), 1);
                const int y2 = min(max(p2, 0), 1), y3 = min(max(p3, 0), 1);
                const uint32_t yn = (uint32_t)(y0 | (y1 << 1) | (y2 << 2) | (y3 << 3));
                const uint32_t hb = ((yh4 * 0x01020408u) >> 24) & 0xFu;   // 0/1 bytes -> bits 0..3
                ss += __popc(hb ^ yn);
                // y changed iff 2*y_new != old y2 (old y2 = 1, i.e. 1/2, on the first pass)
                const uint32_t o2 = (uint32_t)(yo.x | (yo.y << 2) | (yo.z << 4) | (yo.w << 6));
                const uint32_t n2 = (uint32_t)((y0 << 1) | (y1 << 3) | (y2 << 5) | (y3 << 7));
                const bool ychg = o2 != n2;
                chg_self |= ychg | (hb != yn);
                const int go = goff_[j];
                __stcs(reinterpret_cast<int4 *>(a_t + go),
                       make_int4(av.x + h0 - y0, av.y + h1 - y1, av.z + h2 - y2, av.w + h3 - y3));
                __stcg(reinterpret_cast<int4 *>(y_t + go), make_int4(2 * y0, 2 * y1, 2 * y2, 2 * y3));
                if (ychg) {
                    chgU |= top;
                    chgD |= bot;
                    chgL |= lft && ((o2 & 3u) != (n2 & 3u));
                    chgR |= rgt && ((o2 >> 6) != (n2 >> 6));
                }
            }
            // every warp is done with stage s: refill it with the tile STAGES ahead
            __syncthreads();
            if (tid == 0 && ikb < nblk) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                int by2, bx2;
                coords(ikb, by2, bx2);
                tma_issue_tile<TW>(L, M, base + s * C::STAGE, &full[s], by2, bx2, itile, cur, p);
                if (++itile == tpb) { itile = 0; ++ikb; }
            }
            if (++s == C::STAGES) { s = 0; phase ^= 1u; }
        }
        // publish this block's partials: one atomic per warp
        const int64_t e = warp_sum(e_acc + (int64_t)L.lamw * quad_acc);
        const int sq = warp_sum(ss);
        const unsigned fl = __ballot_sync(FULLMASK, clamped), f0 = __ballot_sync(FULLMASK, chg_self),
                       f1 = __ballot_sync(FULLMASK, chgL), f2 = __ballot_sync(FULLMASK, chgR),
                       f3 = __ballot_sync(FULLMASK, chgU), f4 = __ballot_sync(FULLMASK, chgD);
        if (lane == 0) {
            if (e) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pe[k]), (unsigned long long)e);
            if (sq) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pr[k]), (unsigned long long)sq);
            if (fl) atomicOr(&L.pf[k], 1);
            if (f0) L.dirty[k] = 1u;
            if (f1) L.dirty[k - 1] = 1u;
            if (f2) L.dirty[k + 1] = 1u;
            if (f3 && k - KX >= 0) L.dirty[k - KX] = 1u;
            if (f4 && k + KX < L.K) L.dirty[k + KX] = 1u;
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const int prev = atomicAdd(&st->done_ctas, 1);
        last = (prev == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        finalize_cta(L, cur, best, out);
        __syncthreads();
        // partials were accumulated: clear them for the next iteration
        for (int k = tid; k < L.K; k += blockDim.x) {
            L.pe[k] = 0;
            L.pr[k] = 0;
            L.pf[k] = 0;
        }
        if (tid == 0) st->done_ctas = 0;
    }
}
