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

template <int TW>
struct TmaCfg {
    static constexpr int TH = 4096 / TW;                 // tile rows (64 or 32)
    static constexpr int NT = 256;
    static constexpr int QPT = TH * TW / 4 / NT;         // quads per thread (4)
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
    static constexpr int STAGES = 3;
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
                                               uint64_t *bar, int k, int tile, int cur, int p) {
    using C = TmaCfg<TW>;
    const int by = k / L.ax.k, bx = k - by * L.ax.k;
    const int x0 = bx * TW;                       // uniform tiling: lo = index * width
    const int y0 = by * L.ay.base + tile * C::TH;
    mbar_expect_tx(bar, C::TX);
    tma_load_2d(stage + C::O_U, &M.u, bar, x0, y0);
    tma_load_2d(stage + C::O_A, &M.a[p], bar, x0, y0);
    tma_load_2d(stage + C::O_Y, &M.y[cur], bar, x0, y0);
    tma_load_2d(stage + C::O_YR, &M.yr[cur], bar, x0 + TW, y0);
    tma_load_2d(stage + C::O_H, &M.yhat, bar, x0 - 16, y0 - 1);
}

template <int TW>
__global__ void __launch_bounds__(256, 1) k_consensus_tma(Lat2 L, const __grid_constant__ TmaMaps M) {
    using C = TmaCfg<TW>;
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
    const int32_t W = L.W, H = L.ay.dim, q = L.q, BH = L.ay.base;
    const int tiles_per_block = BH / TH;
    const int nblk = (L.K - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int ntiles = nblk * tiles_per_block;

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < C::STAGES && i < ntiles; ++i) {
            const int k = blockIdx.x + (i / tiles_per_block) * gridDim.x;
            tma_issue_tile<TW>(L, M, base + i * C::STAGE, &full[i], k, i % tiles_per_block, cur, p);
        }
    }
    __syncthreads();

    int64_t e_acc = 0, ss = 0;
    int quad_acc = 0, clamped = 0, chg_self = 0, chgL = 0, chgR = 0, chgU = 0, chgD = 0;
    for (int i = 0; i < ntiles; ++i) {
        const int s = i % C::STAGES;
        const int k = blockIdx.x + (i / tiles_per_block) * gridDim.x;
        const int tile = i % tiles_per_block;
        const int by = k / L.ax.k, bx = k - by * L.ax.k;
        const int lo_r = by * BH, lo_c = bx * TW;
        const int r0 = tile * TH;                      // first block row of this tile
        const bool has_up = lo_r > 0, has_dn = lo_r + BH < H, has_lf = lo_c > 0, has_rt = lo_c + TW < W;
        uint8_t *sb = base + s * C::STAGE;
        const int32_t *su = reinterpret_cast<const int32_t *>(sb + C::O_U);
        const int32_t *sa = reinterpret_cast<const int32_t *>(sb + C::O_A);
        const int32_t *sy = reinterpret_cast<const int32_t *>(sb + C::O_Y);
        const int32_t *syr = reinterpret_cast<const int32_t *>(sb + C::O_YR);
        const uint8_t *sh = sb + C::O_H;
        mbar_wait(&full[s], (uint32_t)((i / C::STAGES) & 1));

#pragma unroll
        for (int j = 0; j < QPT; ++j) {
            const int t = tid + j * NT;
            const int rr = t >> LQ, c0 = (t & (QR - 1)) << 2;   // row within tile
            const int r = r0 + rr;                               // row within block
            const int4 av = *reinterpret_cast<const int4 *>(sa + rr * TW + c0);
            const int4 yo = *reinterpret_cast<const int4 *>(sy + rr * TW + c0);
            const int4 uu = *reinterpret_cast<const int4 *>(su + rr * TW + c0);
            const uint32_t yh4 = *reinterpret_cast<const uint32_t *>(sh + (rr + 1) * C::YHW + 16 + c0);
            const uint32_t ob = (uint32_t)((yo.x >> 1) | ((yo.y >> 1) << 1) | ((yo.z >> 1) << 2) |
                                           ((yo.w >> 1) << 3));
            const uint32_t nxt = __shfl_down_sync(FULLMASK, ob, 1);
            const bool top = (r == 0 && has_up), bot = (r == BH - 1 && has_dn);
            const bool lft = (c0 == 0 && has_lf), rgt = (c0 + 4 == TW && has_rt);
            if (want_e) {
                const int4 yb = *reinterpret_cast<const int4 *>(sy + (rr + 1) * TW + c0);
                const uint32_t bb = (uint32_t)((yb.x >> 1) | ((yb.y >> 1) << 1) | ((yb.z >> 1) << 2) |
                                               ((yb.w >> 1) << 3));
                int qd = __popc((ob ^ (ob >> 1)) & 0x7u);
                if (c0 + 4 < TW) qd += (int)((ob >> 3) ^ (nxt & 1u));
                else if (has_rt) qd += (int)((ob >> 3) ^ (uint32_t)(syr[rr * 4] >> 1));
                if (lo_r + r + 1 < H) qd += __popc(ob ^ bb);
                quad_acc += qd;
                e_acc += (ob & 1u ? uu.x : 0) + (ob & 2u ? uu.y : 0) + (ob & 4u ? uu.z : 0) +
                         (ob & 8u ? uu.w : 0);
            }
            const uint32_t up4 = *reinterpret_cast<const uint32_t *>(sh + rr * C::YHW + 16 + c0);
            const uint32_t dn4 = *reinterpret_cast<const uint32_t *>(sh + (rr + 2) * C::YHW + 16 + c0);
            const int lfb = sh[(rr + 1) * C::YHW + 15 + c0];
            const int rtb = sh[(rr + 1) * C::YHW + 20 + c0];
            const int a4[4] = {av.x, av.y, av.z, av.w};
            const int y24[4] = {yo.x, yo.y, yo.z, yo.w};
            int y[4], an[4];
            bool ychg_any = false;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int yh = byte_of(yh4, e);
                int sx = 0;
                if (top) sx += yh - byte_of(up4, e);
                if (bot) sx += yh - byte_of(dn4, e);
                if (e == 0 && lft) sx += yh - lfb;
                if (e == 3 && rgt) sx += yh - rtb;
                const int ypre = yh + a4[e] - q * sx;
                clamped |= (unsigned)ypre > 1u;
                y[e] = ypre < 0 ? 0 : (ypre > 1 ? 1 : ypre);
                an[e] = a4[e] + yh - y[e];
                ss += yh ^ y[e];
                const bool ychg = (2 * y[e] != y24[e]);
                ychg_any |= ychg;
                chg_self |= ychg | (yh != y[e]);
            }
            const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c0;
            __stcs(reinterpret_cast<int4 *>(a_out + G), make_int4(an[0], an[1], an[2], an[3]));
            __stcg(reinterpret_cast<int4 *>(y_out + G), make_int4(2 * y[0], 2 * y[1], 2 * y[2], 2 * y[3]));
            if (ychg_any) {
                chgU |= top;
                chgD |= bot;
                chgL |= (lft && (2 * y[0] != y24[0]));
                chgR |= (rgt && (2 * y[3] != y24[3]));
            }
        }
        // every warp is done with stage s: refill it with tile i + STAGES
        __syncthreads();
        if (tid == 0 && i + C::STAGES < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int i2 = i + C::STAGES;
            const int k2 = blockIdx.x + (i2 / tiles_per_block) * gridDim.x;
            tma_issue_tile<TW>(L, M, base + s * C::STAGE, &full[s], k2, i2 % tiles_per_block, cur, p);
        }
        if (tile == tiles_per_block - 1) {
            // publish this block's partials: one atomic per warp
            const int64_t e = warp_sum(e_acc + (int64_t)L.lamw * quad_acc);
            const int64_t sq = warp_sum(ss);
            const bool fl = __any_sync(FULLMASK, clamped);
            const bool f0 = __any_sync(FULLMASK, chg_self), f1 = __any_sync(FULLMASK, chgL),
                       f2 = __any_sync(FULLMASK, chgR), f3 = __any_sync(FULLMASK, chgU),
                       f4 = __any_sync(FULLMASK, chgD);
            if (lane == 0) {
                if (e) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pe[k]), (unsigned long long)e);
                if (sq) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pr[k]), (unsigned long long)sq);
                if (fl) atomicOr(&L.pf[k], 1);
                if (f0) L.dirty[k] = 1u;
                if (f1) L.dirty[k - 1] = 1u;
                if (f2) L.dirty[k + 1] = 1u;
                if (f3) L.dirty[k - L.ax.k] = 1u;
                if (f4) L.dirty[k + L.ax.k] = 1u;
            }
            e_acc = 0; ss = 0; quad_acc = 0; clamped = 0;
            chg_self = chgL = chgR = chgU = chgD = 0;
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
