// lattice3d.cuh -- 3D 6-connected lattices (BASELINE C4: 256^3, 32^3 sub-regions).
// Included by dope_lattice.cu inside namespace dope.
//
// Same algorithm and exactness argument as the 2D kernels; the
// difference is where the block's residual graph lives.  A 32^3 sub-region has
// 32768 nodes and 6 arcs per node: excess (int32) + 6 residual bytes + height
// (uint16) is 12 B/node = 384 KB, more than one SM's shared memory.  K1-3D
// therefore keeps the node state in a per-sub-region HBM scratch that stays
// L2-resident while the CTA works on it (32 MB for 148 resident blocks vs the
// 126 MB L2); only the BFS bit masks (8 x 4 KB) live in shared memory, where
// one warp runs the bit-parallel global relabel with +-1 / +-BW / +-BW*BH word
// shifts.  Residual planes double as the warm-start state (no copies).

struct Geo3 {
    int32_t lo_z, dz, lo_r, hr, lo_c, wc;
};

__device__ __forceinline__ Geo3 block_geo3(const Lat2 &L, int k, int &bz, int &by, int &bx) {
    const int kyx = L.ay.k * L.ax.k;
    bz = k / kyx;
    const int rem = k - bz * kyx;
    by = rem / L.ax.k;
    bx = rem - by * L.ax.k;
    Geo3 g;
    L.az.range(bz, g.lo_z, g.dz);
    L.ay.range(by, g.lo_r, g.hr);
    L.ax.range(bx, g.lo_c, g.wc);
    return g;
}

template <int BD, int BH, int BW, int NT>
struct K1Cfg3 {
    static constexpr int M = BD * BH * BW;
    static constexpr int PL = BH * BW;
    static_assert(M % NT == 0 && M % 64 == 0, "layout");
    static constexpr int NPT = M / NT;
    static constexpr int NW = M / 64;
    static constexpr size_t SMEM = (size_t)9 * 8 * NW + 64;   // 8 masks + reach + misc
};

// Solve of sub-region k with its node state in the per-block HBM scratch.
// The E, S, D residual planes (0, 2, 4) are the persistent truth between
// solves; a warm start re-derives W, N, U (r(v->v-off) = 2cap - r(v-off->v))
// so the shared-memory kernel below, which stores only E/S/D, and this one
// can alternate on the same block.
template <int BD, int BH, int BW, int NT>
__device__ __forceinline__ void mincut3d_l2(const Lat2 &L, const K1Tune &T, int k, uint8_t *smem3) {
    using C = K1Cfg3<BD, BH, BW, NT>;
    constexpr int M = C::M, NPT = C::NPT, NW = C::NW, PL = C::PL;
    uint64_t *masks = reinterpret_cast<uint64_t *>(smem3);   // E W S N D U SINK ACT
    uint64_t *reach = masks + 8 * NW;
    int *misc = reinterpret_cast<int *>(reach + NW);
    uint32_t *masks32 = reinterpret_cast<uint32_t *>(masks);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    int bz, by, bx;
    const Geo3 gb = block_geo3(L, k, bz, by, bx);
    const int32_t W = L.W, H = L.ay.dim, D = L.az.dim;
    const int64_t HW = (int64_t)H * W;
    const int32_t cap = L.cap;
    const astore_t *__restrict__ a_cur = L.a;
    const ystore_t *__restrict__ y_cur = L.y2[L.st->ycur];
    int32_t *g = reinterpret_cast<int32_t *>(L.scratch + (size_t)k * 6 * M);
    uint16_t *h = reinterpret_cast<uint16_t *>(g + M);
    uint8_t *rr = L.resid + (size_t)k * 6 * M;
    const bool up_z = gb.lo_z > 0 || L.gzu, dn_z = gb.lo_z + gb.dz < D || L.gzd;   // ghost planes: shards
    const bool up_r = gb.lo_r > 0, dn_r = gb.lo_r + gb.hr < H;
    const bool lf_c = gb.lo_c > 0, rt_c = gb.lo_c + gb.wc < W;

    // ---- prologue: 2*linear on the 6-neighbour cross-block stencil ----
#pragma unroll 4
    for (int i = 0; i < NPT; ++i) {
        const int v = tid + i * NT;
        const int z = v / PL, r = (v / BW) % BH, c = v % BW;
        const bool valid = z < gb.dz && r < gb.hr && c < gb.wc;
        int32_t gv = 0;
        if (valid) {
            const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + r) * W + gb.lo_c + c;
            const int32_t yg = (int32_t)y_cur[G];
            int32_t sx = 0;
            if (c == 0 && lf_c) sx += yg - y_cur[G - 1];
            if (c == gb.wc - 1 && rt_c) sx += yg - y_cur[G + 1];
            if (r == 0 && up_r) sx += yg - y_cur[G - W];
            if (r == gb.hr - 1 && dn_r) sx += yg - y_cur[G + W];
            if (z == 0 && up_z) sx += yg - y_cur[G - HW];
            if (z == gb.dz - 1 && dn_z) sx += yg - y_cur[G + HW];
            const int32_t lin2 = 2 * L.u[G] + L.lamw * sx + L.mu * (2 * (int32_t)a_cur[G] - yg) + L.mu;
            const bool has[6] = {c + 1 < gb.wc, c > 0, r + 1 < gb.hr, r > 0, z + 1 < gb.dz, z > 0};
            if (L.warm) {
                int32_t f = 0;
#pragma unroll
                for (int d = 0; d < 6; ++d) {
                    if (!has[d]) continue;
                    int32_t r;
                    if (d & 1) {   // reverse arc: from the forward plane of the neighbour
                        const int off = d == 1 ? 1 : d == 3 ? BW : PL;
                        r = 2 * cap - (int32_t)rr[(d - 1) * M + v - off];
                        rr[d * M + v] = (uint8_t)r;
                    } else {
                        r = rr[d * M + v];
                    }
                    f += r - cap;
                }
                gv = lin2 + f;
            } else {
#pragma unroll
                for (int d = 0; d < 6; ++d) rr[d * M + v] = has[d] ? (uint8_t)cap : 0;
                gv = lin2;
            }
        } else if (!L.warm) {
#pragma unroll
            for (int d = 0; d < 6; ++d) rr[d * M + v] = 0;
        }
        g[v] = gv;
    }
    __syncthreads();

    int rounds = 0;
    long long sweeps_done = 0;
    for (;;) {
#pragma unroll 2
        for (int i = 0; i < NPT; ++i) {
            const int v = tid + i * NT;
            const int32_t gv = g[v];
            uint32_t b[6];
#pragma unroll
            for (int d = 0; d < 6; ++d) b[d] = __ballot_sync(FULLMASK, rr[d * M + v] != 0);
            const uint32_t bK = __ballot_sync(FULLMASK, gv < 0);
            const uint32_t bA = __ballot_sync(FULLMASK, gv > 0);
            h[v] = gv < 0 ? 0 : HINF;
            if (lane == 0) {
                const int w32 = (i * NT + warp * 32) >> 5;
#pragma unroll
                for (int d = 0; d < 6; ++d) masks32[d * 2 * NW + w32] = b[d];
                masks32[6 * 2 * NW + w32] = bK;
                masks32[7 * 2 * NW + w32] = bA;
            }
        }
        __syncthreads();
        if (warp == 0) {
            int levels = 0;
            const int hit = bfs_relabel<NW, BW, PL>(masks, reach, h, lane, &levels);
            if (lane == 0) { misc[0] = hit; misc[1] = levels; }
        }
        __syncthreads();
        const int hit = misc[0];
        const int levels = misc[1];
        if (!hit) break;
        if (++rounds > T.max_rounds) {
            if (tid == 0) atomicCAS(&L.st->error, 0, k + 1);
            break;
        }
        const int cap_sweeps = T.sweep_min + T.sweep_mul * levels;
        for (int sw = 0; sw < cap_sweeps; ++sw) {
            ++sweeps_done;
#pragma unroll 4
            for (int i = 0; i < NPT; ++i) {
                const int v = tid + i * NT;
                const int32_t e = g[v];
                if (e <= 0) continue;
                const uint16_t hv = h[v];
                if (hv == HINF || hv == 0) continue;
                const uint16_t ht = hv - 1;
                int32_t left = e;
#pragma unroll
                for (int d = 0; d < 6; ++d) {
                    const int off = (d == 0) ? 1 : (d == 1) ? -1 : (d == 2) ? BW : (d == 3) ? -BW
                                  : (d == 4) ? PL : -PL;
                    const int32_t rv = rr[d * M + v];
                    if (rv == 0) continue;
                    const int w = v + off;
                    if (h[w] != ht) continue;
                    const int32_t delta = left < rv ? left : rv;
                    rr[d * M + v] = (uint8_t)(rv - delta);
                    rr[(d ^ 1) * M + w] = (uint8_t)(rr[(d ^ 1) * M + w] + delta);
                    atomicAdd(&g[w], delta);
                    left -= delta;
                    if (left == 0) break;
                }
                if (left != e) atomicSub(&g[v], e - left);
            }
            __syncthreads();
            int act = 0;
#pragma unroll 4
            for (int i = 0; i < NPT; ++i) {
                const int v = tid + i * NT;
                if (g[v] <= 0) continue;
                const uint16_t hv = h[v];
                if (hv == HINF) continue;
                uint32_t mn = HINF;
#pragma unroll
                for (int d = 0; d < 6; ++d) {
                    const int off = (d == 0) ? 1 : (d == 1) ? -1 : (d == 2) ? BW : (d == 3) ? -BW
                                  : (d == 4) ? PL : -PL;
                    if (rr[d * M + v] == 0) continue;
                    const uint32_t hw = h[v + off];
                    mn = hw < mn ? hw : mn;
                }
                const uint32_t nh = (mn + 1 >= (uint32_t)M) ? HINF : mn + 1;
                if (nh != hv) h[v] = (uint16_t)nh;
                act |= (nh != HINF);
            }
            if (!__syncthreads_or(act)) break;
        }
    }
    // ---- epilogue: labels (sink side); the residual planes stay in place ----
    for (int i = 0; i < NPT; ++i) {
        const int v = tid + i * NT;
        const int z = v / PL, r = (v / BW) % BH, c = v % BW;
        if (z < gb.dz && r < gb.hr && c < gb.wc) {
            const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + r) * W + gb.lo_c + c;
            L.yhat[G] = (uint8_t)((reach[v >> 6] >> (v & 63)) & 1ull);
        }
    }
    if (tid == 0) {
        atomicAdd((unsigned long long *)&L.st->solves, 1ull);
        atomicAdd((unsigned long long *)&L.st->sweeps, (unsigned long long)sweeps_done);
        atomicMax(&L.st->max_rounds_seen, rounds);
    }
}

template <int BD, int BH, int BW, int NT>
__global__ void __launch_bounds__(NT) k_block_mincut3d(Lat2 L, K1Tune T) {
    extern __shared__ __align__(16) uint8_t smem3[];
    const int k = blockIdx.x;
    if (L.st->stop || (L.skip_clean && L.dirty[k] == 0)) {
        if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        L.dirty[k] = 0;
        L.dirty[L.K + k] = (uint32_t)L.st->iteration + 1u;   // solve epoch
    }
    mincut3d_l2<BD, BH, BW, NT>(L, T, k, smem3);
    if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
}

__global__ void k_init_resid3d(Lat2 L, int boxd, int boxh, int boxw) {
    const int k = blockIdx.x;
    const int M = boxd * boxh * boxw, PL = boxh * boxw;
    int bz, by, bx;
    const Geo3 gb = block_geo3(L, k, bz, by, bx);
    uint8_t *gres = L.resid + (size_t)k * 6 * M;
    for (int v = threadIdx.x; v < M; v += blockDim.x) {
        const int z = v / PL, r = (v / boxw) % boxh, c = v % boxw;
        const bool valid = z < gb.dz && r < gb.hr && c < gb.wc;
        const bool has[6] = {c + 1 < gb.wc, c > 0, r + 1 < gb.hr, r > 0, z + 1 < gb.dz, z > 0};
        for (int d = 0; d < 6; ++d) gres[d * M + v] = (valid && has[d]) ? (uint8_t)L.cap : 0;
    }
}

// Consensus for 3D (scalar, one CTA per sub-region).  Same semantics as
// k_consensus: y_t into the free buffer, multipliers, residual partials,
// energy partials of y_{t-1}, dirty marks for the block and its 6 face
// neighbours, last-CTA finalize.
__global__ void __launch_bounds__(512) k_consensus3d(Lat2 L) {
    if (L.st->stop) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = blockIdx.x;
    int bz, by, bx;
    const Geo3 gb = block_geo3(L, k, bz, by, bx);
    const int32_t W = L.W, H = L.ay.dim, D = L.az.dim;
    const int64_t HW = (int64_t)H * W;
    const int cur = L.st->ycur, best = L.st->ybest, out = other_buffer(cur, best);
    const ystore_t *__restrict__ y_in = L.y2[cur];
    ystore_t *__restrict__ y_out = L.y2[out];
    // multipliers are updated in place (a_{t+1}[p] depends on a_t[p] only)
    const astore_t *a_in = L.a;
    astore_t *a_out = L.fuse ? L.a : nullptr;
    const bool want_e = L.fuse && L.st->iteration >= 1;
    const bool up_z = gb.lo_z > 0 || L.gzu, dn_z = gb.lo_z + gb.dz < D || L.gzd;   // ghost planes: shards
    const bool up_r = gb.lo_r > 0, dn_r = gb.lo_r + gb.hr < H;
    const bool lf_c = gb.lo_c > 0, rt_c = gb.lo_c + gb.wc < W;

    int64_t e_acc = 0, ss = 0, du = 0;
    int clamped = 0;
    unsigned marks = 0;    // bit0 self, 1..6: -x +x -y +y -z +z neighbours
    const int m = gb.dz * gb.hr * gb.wc, pl = gb.hr * gb.wc;
    for (int v = tid; v < m; v += blockDim.x) {
        const int z = v / pl, rem = v - z * pl, r = rem / gb.wc, c = rem - r * gb.wc;
        const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + r) * W + gb.lo_c + c;
        const int32_t yh = L.yhat[G];
        int32_t sx = 0;
        if (c == 0 && lf_c) sx += yh - L.yhat[G - 1];
        if (c == gb.wc - 1 && rt_c) sx += yh - L.yhat[G + 1];
        if (r == 0 && up_r) sx += yh - L.yhat[G - W];
        if (r == gb.hr - 1 && dn_r) sx += yh - L.yhat[G + W];
        if (z == 0 && up_z) sx += yh - L.yhat[G - HW];
        if (z == gb.dz - 1 && dn_z) sx += yh - L.yhat[G + HW];
        const int32_t aold = (int32_t)a_in[G];
        const int32_t ypre = yh + aold - L.q * sx;
        const int32_t y = ypre < 0 ? 0 : (ypre > 1 ? 1 : ypre);
        const int32_t y2old = (int32_t)y_in[G];
        clamped |= (ypre < 0 || ypre > 1);
        if (a_out) a_out[G] = (astore_t)(aold + yh - y);
        y_out[G] = (ystore_t)(2 * y);
        ss += (yh - y) * (yh - y);
        if (want_e) {
            const int32_t o = y2old >> 1;
            int32_t qd = 0;
            const int gc = gb.lo_c + c, gr = gb.lo_r + r, gz = gb.lo_z + z;
            if (gc + 1 < W) qd += o ^ (y_in[G + 1] >> 1);
            if (gr + 1 < H) qd += o ^ (y_in[G + W] >> 1);
            if (gz + 1 < D || L.gzd) qd += o ^ (y_in[G + HW] >> 1);
            e_acc += (int64_t)L.lamw * qd;
        }
        const bool ychg = (2 * y != y2old);
        if (ychg || yh != y) marks |= 1u;
        if (ychg) {
            marks |= 256u;
            du += (int64_t)L.u[G] * (2 * y - y2old);
            if (c == 0 && lf_c) marks |= 2u;
            if (c == gb.wc - 1 && rt_c) marks |= 4u;
            if (r == 0 && up_r) marks |= 8u;
            if (r == gb.hr - 1 && dn_r) marks |= 16u;
            if (z == 0 && up_z) marks |= 32u;
            if (z == gb.dz - 1 && dn_z) marks |= 64u;
        }
    }
    __shared__ int64_t red_e[32], red_s[32], red_u[32];
    __shared__ unsigned red_f[32];
    e_acc = warp_sum(e_acc);
    ss = warp_sum(ss);
    du = warp_sum(du);
    for (int o = 16; o > 0; o >>= 1) marks |= __shfl_xor_sync(FULLMASK, marks, o);
    const int fl = __any_sync(FULLMASK, clamped);
    if (lane == 0) { red_e[warp] = e_acc; red_s[warp] = ss; red_u[warp] = du; red_f[warp] = marks | (fl ? 128u : 0u); }
    __syncthreads();
    if (tid == 0) {
        int64_t E = 0, S = 0, U = 0;
        unsigned Fm = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { E += red_e[w]; S += red_s[w]; U += red_u[w]; Fm |= red_f[w]; }
        L.pe[k] = E;
        L.pu[k] = U;
        L.pr[k] = S;
        L.pf[k] = (Fm & 128u) ? 1 : 0;
        const int KX = L.ax.k, KYX = L.ay.k * L.ax.k;
        if (Fm & 1u) mark_dirty(L, k);
        if (Fm & 2u) mark_dirty(L, k - 1);
        if (Fm & 4u) mark_dirty(L, k + 1);
        if (Fm & 8u) mark_dirty(L, k - KX);
        if (Fm & 16u) mark_dirty(L, k + KX);
        if ((Fm & 32u) && k - KYX >= 0) mark_dirty(L, k - KYX);
        if ((Fm & 64u) && k + KYX < L.K) mark_dirty(L, k + KYX);
        ybuf_stamp(L, out)[k] = (uint32_t)L.st->iteration + 1u;
        if (Fm & 256u) ychg_stamp(L)[k] = (uint32_t)L.st->iteration + 1u;
        CtaAgg agg;
        agg.add_block(E, U, S, (Fm & 128u) ? 1 : 0);
        pass_tail(L, agg, cur, best, out);
    }
}

// Vectorised 3D consensus (blocks whose x extent is a multiple of 4 on a grid
// whose width is too): thread t owns quads of 4 consecutive x voxels; the
// quads of one block row sit in consecutive lanes, so the energy's +x pair of
// a quad's last voxel comes from the next lane.  Loads are issued in batches
// of 4 quads before any is used.  Persistent over blocks; same arithmetic as
// k_consensus3d.
template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) k_consensus3d_vec(Lat2 L, int lq) {
    constexpr int QB = 4;   // quads per load batch
    if (L.pdl) {
        griddep_wait();
        griddep_launch();
    }
    if (L.st->stop) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    CtaAgg agg;
    const int cur = L.st->ycur, best = L.st->ybest, out = other_buffer(cur, best);
    const ystore_t *__restrict__ y_in = L.y2[cur];
    ystore_t *__restrict__ y_out = L.y2[out];
    const astore_t *a_in = L.a;
    astore_t *a_out = L.fuse ? L.a : nullptr;
    const int it = L.st->iteration;
    const bool want_e = L.fuse && it >= 1;
    // clean-block pass: needs the multipliers updated here, re-solves skipped
    // for unchanged blocks, and energy partials from an earlier pass (it >= 2)
    const bool clean_ok = L.fuse && L.skip_clean && it >= 2;
    const uint32_t ep = (uint32_t)it + 1u;
    const int32_t W = L.W, H = L.ay.dim, D = L.az.dim, q = L.q;
    const int64_t HW = (int64_t)H * W;
    const int QR = 1 << lq;
    __shared__ int64_t red_e[NT / 32], red_s[NT / 32], red_u[NT / 32];
    __shared__ unsigned red_f[NT / 32];
    for (int k = blockIdx.x; k < L.K; k += gridDim.x) {
        int bz, by, bx;
        const Geo3 gb = block_geo3(L, k, bz, by, bx);
        const bool up_z = gb.lo_z > 0 || L.gzu, dn_z = gb.lo_z + gb.dz < D || L.gzd;   // ghost planes: shards
        const bool up_r = gb.lo_r > 0, dn_r = gb.lo_r + gb.hr < H;
        const bool lf_c = gb.lo_c > 0, rt_c = gb.lo_c + gb.wc < W;
        const int nq = (gb.dz * gb.hr) << lq;
        if (clean_ok) {
            // Fixed point: a block K1 did not re-solve had yhat == y and no y
            // change in the previous pass (else it would be dirty); with none
            // of its 6 neighbours re-solved either, every voxel's pre-clamp
            // value repeats: y, a, clamp status, residual 0, and the pair
            // energy of y_{t-1} equals the stored partial.  Only the output
            // buffer may need the block's iterate.
            const int KX = L.ax.k, KYX = L.ay.k * L.ax.k;
            const uint32_t *epo = L.dirty + L.K;
            bool fast = epo[k] != ep;
            fast = fast && !(lf_c && epo[k - 1] == ep) && !(rt_c && epo[k + 1] == ep);
            fast = fast && !(up_r && epo[k - KX] == ep) && !(dn_r && epo[k + KX] == ep);
            fast = fast && !(gb.lo_z > 0 && epo[k - KYX] == ep) && !(gb.lo_z + gb.dz < D && epo[k + KYX] == ep);
            fast = fast && !(gb.lo_z == 0 && L.gzu) && !(gb.lo_z + gb.dz == D && L.gzd);   // other rank's solves unknown
            if (fast) {
                const uint32_t st_out = ybuf_stamp(L, out)[k];
                if (st_out == 0u || st_out < ychg_stamp(L)[k]) {
                    for (int t = tid; t < nq; t += NT) {
                        const int row = t >> lq, c0 = (t & (QR - 1)) << 2;
                        const int z = row / gb.hr, r = row - z * gb.hr;
                        const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + r) * W + gb.lo_c + c0;
                        __stcg(reinterpret_cast<unsigned int *>(y_out + G),
                               __ldcg(reinterpret_cast<const unsigned int *>(y_in + G)));
                    }
                }
                __syncthreads();   // every thread has read the stamps
                if (tid == 0) {
                    ybuf_stamp(L, out)[k] = ep;
                    L.pu[k] = 0;
                    L.pr[k] = 0;
                    agg.add_block(L.pe[k], 0, 0, L.pf[k]);
                }
                continue;
            }
        }
        int64_t e_acc = 0, du = 0;
        int ss = 0;
        unsigned marks = 0, clamp_or = 0;   // marks: bit0 self, 1..6 -x +x -y +y -z +z
        for (int t0 = 0; t0 < nq; t0 += QB * NT) {
            uint32_t yh4[QB], yo[QB], nb[QB], cnt[QB], yb[QB], yz[QB];
            uint2 av[QB];
            int yr[QB];
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                const int t = t0 + tid + j * NT;
                yh4[j] = yo[j] = nb[j] = cnt[j] = yb[j] = yz[j] = 0;
                av[j] = make_uint2(0, 0);
                yr[j] = 0;
                if (t < nq) {
                    const int row = t >> lq, c0 = (t & (QR - 1)) << 2;
                    const int z = row / gb.hr, r = row - z * gb.hr;
                    const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + r) * W + gb.lo_c + c0;
                    yh4[j] = __ldcs(reinterpret_cast<const unsigned int *>(L.yhat + G));
                    av[j] = __ldcs(reinterpret_cast<const uint2 *>(a_in + G));
                    yo[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G));
                    if (want_e) {
                        if (gb.lo_r + r + 1 < H) yb[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G + W));
                        if (gb.lo_z + z + 1 < D || L.gzd) yz[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G + HW));
                        if (c0 + 4 == gb.wc && gb.lo_c + c0 + 4 < W) yr[j] = y_in[G + 4];
                    }
                    // cross-block neighbour labels: count / sum per voxel (bytes)
                    if (r == 0 && up_r) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G - W); }
                    if (r == gb.hr - 1 && dn_r) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G + W); }
                    if (z == 0 && up_z) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G - HW); }
                    if (z == gb.dz - 1 && dn_z) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G + HW); }
                    if (c0 == 0 && lf_c) { cnt[j] += 1u; nb[j] += L.yhat[G - 1]; }
                    if (c0 + 4 == gb.wc && rt_c) { cnt[j] += 1u << 24; nb[j] += (uint32_t)L.yhat[G + 4] << 24; }
                }
            }
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                const int t = t0 + tid + j * NT;
                const uint32_t nxt = __shfl_down_sync(FULLMASK, yo[j], 1);
                if (t >= nq) continue;
                const int row = t >> lq, c0 = (t & (QR - 1)) << 2;
                const int z = row / gb.hr, r = row - z * gb.hr;
                const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + r) * W + gb.lo_c + c0;
                if (want_e) {
                    // y2 bytes are 0/2: each differing pair is one set bit of the XOR
                    uint32_t rw;
                    if (c0 + 4 < gb.wc) rw = nxt;
                    else rw = (gb.lo_c + c0 + 4 < W) ? (uint32_t)yr[j] : (yo[j] >> 24);
                    int qd = __popc(yo[j] ^ __funnelshift_r(yo[j], rw, 8));
                    if (gb.lo_r + r + 1 < H) qd += __popc(yo[j] ^ yb[j]);
                    if (gb.lo_z + z + 1 < D || L.gzd) qd += __popc(yo[j] ^ yz[j]);
                    e_acc += (int64_t)L.lamw * qd;
                }
                // y = clamp(h + a - q*sx), sx = cnt*h - nb (biased by 4)
                const uint32_t h4 = yh4[j];
                const uint32_t sb = ((cnt[j] & (h4 * 0xFFu)) | 0x04040404u) - nb[j];
                int a4[4];
                unpack_a4(av[j], a4);
                int y[4], an[4];
                uint32_t yw = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int h = (int)((h4 >> (8 * i)) & 0xFFu);
                    const int p = a4[i] + h + 4 * q - q * (int)((sb >> (8 * i)) & 0xFFu);
                    clamp_or |= (uint32_t)p;
                    y[i] = p > 0 ? 1 : 0;
                    an[i] = a4[i] + h - y[i];
                    ss += h ^ y[i];
                    yw |= (uint32_t)(2 * y[i]) << (8 * i);
                }
                if (a_out) __stcs(reinterpret_cast<uint2 *>(a_out + G), pack_a4(an[0], an[1], an[2], an[3]));
                __stcg(reinterpret_cast<unsigned int *>(y_out + G), yw);
                const uint32_t chg = yw ^ yo[j];
                const uint32_t hb = ((h4 * 0x01020408u) >> 24) & 0xFu;
                const uint32_t yb4 = (uint32_t)(y[0] | (y[1] << 1) | (y[2] << 2) | (y[3] << 3));
                if (chg | (hb ^ yb4)) marks |= 1u;
                if (chg) {
                    marks |= 256u;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int dy = (int)((yw >> (8 * i)) & 0xFFu) - (int)((yo[j] >> (8 * i)) & 0xFFu);
                        if (dy) du += (int64_t)__ldg(L.u + G + i) * dy;
                    }
                    if (c0 == 0 && lf_c && (chg & 0xFFu)) marks |= 2u;
                    if (c0 + 4 == gb.wc && rt_c && (chg >> 24)) marks |= 4u;
                    if (r == 0 && up_r) marks |= 8u;
                    if (r == gb.hr - 1 && dn_r) marks |= 16u;
                    if (z == 0 && up_z) marks |= 32u;
                    if (z == gb.dz - 1 && dn_z) marks |= 64u;
                }
            }
        }
        // block reduction
        e_acc = warp_sum(e_acc);
        du = warp_sum(du);
        const int sq = (int)__reduce_add_sync(FULLMASK, (unsigned)ss);
        const unsigned fm = __reduce_or_sync(FULLMASK, marks | (clamp_or > 1u ? 128u : 0u));
        if (lane == 0) { red_e[warp] = e_acc; red_s[warp] = sq; red_u[warp] = du; red_f[warp] = fm; }
        __syncthreads();
        if (tid == 0) {
            int64_t E = 0, S = 0, U = 0;
            unsigned Fm = 0;
            for (int w = 0; w < NT / 32; ++w) { E += red_e[w]; S += red_s[w]; U += red_u[w]; Fm |= red_f[w]; }
            L.pe[k] = E;
            L.pu[k] = U;
            L.pr[k] = S;
            L.pf[k] = (Fm & 128u) ? 1 : 0;
            const int KX = L.ax.k, KYX = L.ay.k * L.ax.k;
            if (Fm & 1u) mark_dirty(L, k);
            if (Fm & 2u) mark_dirty(L, k - 1);
            if (Fm & 4u) mark_dirty(L, k + 1);
            if (Fm & 8u) mark_dirty(L, k - KX);
            if (Fm & 16u) mark_dirty(L, k + KX);
            if ((Fm & 32u) && k - KYX >= 0) mark_dirty(L, k - KYX);
            if ((Fm & 64u) && k + KYX < L.K) mark_dirty(L, k + KYX);
            ybuf_stamp(L, out)[k] = (uint32_t)it + 1u;
            if (Fm & 256u) ychg_stamp(L)[k] = (uint32_t)it + 1u;
            agg.add_block(E, U, S, (Fm & 128u) ? 1 : 0);
        }
        __syncthreads();
    }
    if (tid == 0) pass_tail(L, agg, cur, best, out);
}

// Per-block slab accumulators of the 3D plane consensus pass: E, U, S,
// marks | group bits << 32, arrival count (5 x 8 bytes in a 64-byte slot after
// the u bricks in L.scratch; zero at allocation, left zeroed after each pass).
__device__ __forceinline__ unsigned long long *slab_acc3(const Lat2 &L, int k) {
    const size_t M = (size_t)L.boxd * L.boxh * L.boxw;
    return reinterpret_cast<unsigned long long *>(L.scratch + (size_t)L.K * (7 * M + 128) + (size_t)k * 64);
}

// Quad groups of a 3D block for the clamp memos (part_flags bits 1-27):
// 3 * 3 * 3 classes by the block side(s) a quad touches per axis (none / low /
// high, only sides with a neighbour); group 0 is the interior.
__device__ __forceinline__ int quad_group3(bool lf, bool rt, bool tp, bool bt, bool zb, bool zt) {
    return (lf ? 1 : (rt ? 2 : 0)) + 3 * (tp ? 1 : (bt ? 2 : 0)) + 9 * (zb ? 1 : (zt ? 2 : 0));
}
// groups touching a side in sd (bit0 -x, 1 +x, 2 -y, 3 +y, 4 -z, 5 +z)
__device__ __forceinline__ unsigned active_groups3(uint32_t sd) {
    unsigned m = 0;
    for (int g = 0; g < 27; ++g) {
        const int xs = g % 3, ys = (g / 3) % 3, zs = g / 9;
        if ((xs == 1 && (sd & 1u)) || (xs == 2 && (sd & 2u)) || (ys == 1 && (sd & 4u)) || (ys == 2 && (sd & 8u)) ||
            (zs == 1 && (sd & 16u)) || (zs == 2 && (sd & 32u)))
            m |= 1u << g;
    }
    return m;
}

// 3D consensus for blocks whose (y, x) face is 32 x 32 (C4's 32^3 tiling):
// thread t owns the quad (r = t / 8, c0 = 4 * (t % 8)) of every z-plane of
// the block, so the per-quad geometry is fixed and planes are visited in
// batches of ZB (all loads of a batch issued first).  The pair energy of
// y_{t-1} takes the +x partner from the next lane, the +y partner from the
// lane 8 up (rows r % 4 != 3) and the +z partner from the same thread's next
// plane, reading memory only across warps / blocks.  Same arithmetic, marks,
// stamps and clean-block pass as k_consensus3d_vec.
#ifndef K2P_ZB
#define K2P_ZB 4
#endif
#ifndef K2P_SLAB
#define K2P_SLAB 32   // planes per work unit of the full update (measured 8 / 16 / 32 on C4: 32)
#endif
#ifndef K2P_MINB
#define K2P_MINB 2
#endif
__global__ void __launch_bounds__(256, K2P_MINB) k_consensus3d_plane(Lat2 L) {
    constexpr int NT = 256, ZB = K2P_ZB;
    if (L.pdl) {
        griddep_wait();
        griddep_launch();
    }
    if (L.st->stop) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = tid >> 3, c0 = (tid & 7) << 2;
    CtaAgg agg;
    const int cur = L.st->ycur, best = L.st->ybest, out = other_buffer(cur, best);
    const ystore_t *__restrict__ y_in = L.y2[cur];
    ystore_t *__restrict__ y_out = L.y2[out];
    const astore_t *a_in = L.a;
    astore_t *a_out = L.fuse ? L.a : nullptr;
    const int it = L.st->iteration;
    const bool want_e = L.fuse && it >= 1;
    const bool clean_ok = L.fuse && L.skip_clean && it >= 2;
    const uint32_t ep = (uint32_t)it + 1u;
    const int32_t W = L.W, H = L.ay.dim, D = L.az.dim, q = L.q;
    const int64_t HW = (int64_t)H * W;
    __shared__ int64_t red_e[NT / 32], red_s[NT / 32], red_u[NT / 32];
    __shared__ unsigned red_f[NT / 32], red_g[NT / 32];
    // work units: (block, slab of K2P_SLAB planes); a block's clean-block
    // pass runs in its slab-0 unit, its full update is split over its slabs
    // (per-block accumulators, the last slab to finish publishes)
    const int nsl = (L.az.base + K2P_SLAB - 1) / K2P_SLAB;
    for (int u = blockIdx.x; u < L.K * nsl; u += gridDim.x) {
        const int k = u / nsl, slab = u - k * nsl;
        int bz, by, bx;
        const Geo3 gb = block_geo3(L, k, bz, by, bx);
        if (slab * K2P_SLAB >= gb.dz) continue;   // ragged last block plane
        const bool up_z = gb.lo_z > 0 || L.gzu, dn_z = gb.lo_z + gb.dz < D || L.gzd;   // ghost planes: shards
        const bool up_r = gb.lo_r > 0, dn_r = gb.lo_r + gb.hr < H;
        const bool lf_c = gb.lo_c > 0, rt_c = gb.lo_c + gb.wc < W;
        const int64_t G0 = ((int64_t)gb.lo_z * H + gb.lo_r + r) * W + gb.lo_c + c0;
        // Clean block (not re-solved): it was left with y == yhat and no
        // moving neighbour face in the last pass, so every quad is a fixed
        // point except those on a face whose neighbour was re-solved now, and
        // its energy partial of y_{t-1} equals the one the last pass stored
        // (DESIGN.md §4).  Ghost planes of another shard count as moved.
        // (a stamp already at ep was written in this pass by the block's
        // clean path -- a full-path block publishes only after all its slabs)
        const uint32_t pst = pe_stamp(L)[k];
        if (clean_ok && L.dirty[L.K + k] != ep && (pst == (uint32_t)it || pst == ep) && !(gb.lo_z == 0 && L.gzu) &&
            !(gb.lo_z + gb.dz == D && L.gzd)) {
            if (slab != 0) continue;
            const int KX = L.ax.k, KYX = L.ay.k * L.ax.k;
            const uint32_t *epo = L.dirty + L.K;
            // re-solved neighbours: bit0 -x, 1 +x, 2 -y, 3 +y, 4 -z, 5 +z
            uint32_t sd = 0;
            if (lf_c && epo[k - 1] == ep) sd |= 1u;
            if (rt_c && epo[k + 1] == ep) sd |= 2u;
            if (up_r && epo[k - KX] == ep) sd |= 4u;
            if (dn_r && epo[k + KX] == ep) sd |= 8u;
            if (gb.lo_z > 0 && epo[k - KYX] == ep) sd |= 16u;
            if (gb.lo_z + gb.dz < D && epo[k + KYX] == ep) sd |= 32u;
            const uint32_t st_out = ybuf_stamp(L, out)[k];
            if (st_out == 0u || st_out < ychg_stamp(L)[k]) {   // the output buffer lacks the block's iterate
                for (int z0 = 0; z0 < gb.dz; z0 += 8) {   // 8 planes of loads in flight
                    uint32_t v[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        v[j] = z0 + j < gb.dz ? *reinterpret_cast<const unsigned int *>(y_in + G0 + (z0 + j) * HW) : 0u;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (z0 + j < gb.dz) *reinterpret_cast<unsigned int *>(y_out + G0 + (z0 + j) * HW) = v[j];
                }
            }
            if (sd == 0) {   // settled: partials, flags and the buffer copy all repeat
                __syncthreads();
                if (tid == 0) {
                    ybuf_stamp(L, out)[k] = ep;
                    pe_stamp(L)[k] = ep;
                    L.pu[k] = 0;
                    L.pr[k] = 0;
                    agg.add_block(L.pe[k], 0, 0, L.pf[k] & 1);
                }
                continue;
            }
            __syncthreads();   // the copy lands before the ring quads overwrite it
            // ring quads: those on a face whose neighbour was re-solved, each
            // once (faces in the order -z +z -y +y -x +x; a quad on an earlier
            // active face is skipped)
            const bool zl_ = (sd & 16u) != 0, zh_ = (sd & 32u) != 0, yl_ = (sd & 4u) != 0, yh_ = (sd & 8u) != 0;
            int64_t du_r = 0;
            int ss_r = 0;
            unsigned marks_r = 0, gfresh = 0;
            auto ring_quad = [&](int rr, int cc, int z) {
                const int64_t G = ((int64_t)(gb.lo_z + z) * H + gb.lo_r + rr) * W + gb.lo_c + cc;
                const bool tp = rr == 0 && up_r, bt = rr == 31 && dn_r, lf = cc == 0 && lf_c, rt = cc == 28 && rt_c;
                const bool zb = z == 0 && up_z, zt = z == gb.dz - 1 && dn_z;
                const uint32_t yo = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G));
                const uint32_t h4 = __ldcg(reinterpret_cast<const unsigned int *>(L.yhat + G));
                const uint2 av = __ldcg(reinterpret_cast<const uint2 *>(a_in + G));
                uint32_t cnt = 0, nb = 0;
                if (tp) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(L.yhat + G - W); }
                if (bt) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(L.yhat + G + W); }
                if (zb) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(L.yhat + G - HW); }
                if (zt) { cnt += 0x01010101u; nb += *reinterpret_cast<const uint32_t *>(L.yhat + G + HW); }
                if (lf) { cnt += 1u; nb += L.yhat[G - 1]; }
                if (rt) { cnt += 1u << 24; nb += (uint32_t)L.yhat[G + 4] << 24; }
                const uint32_t sb = ((cnt & (h4 * 0xFFu)) | 0x04040404u) - nb;
                int a4[4];
                unpack_a4(av, a4);
                int y[4], an[4];
                uint32_t yw = 0, qc = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int h = (int)((h4 >> (8 * i)) & 0xFFu);
                    const int p = a4[i] + h + 4 * q - q * (int)((sb >> (8 * i)) & 0xFFu);
                    qc |= (uint32_t)p;
                    y[i] = p > 0 ? 1 : 0;
                    an[i] = a4[i] + h - y[i];
                    ss_r += h ^ y[i];
                    yw |= (uint32_t)(2 * y[i]) << (8 * i);
                }
                gfresh |= (qc > 1u ? 1u : 0u) << quad_group3(lf, rt, tp, bt, zb, zt);
                __stcs(reinterpret_cast<uint2 *>(a_out + G), pack_a4(an[0], an[1], an[2], an[3]));
                __stcg(reinterpret_cast<unsigned int *>(y_out + G), yw);
                const uint32_t chg = yw ^ yo;
                const uint32_t hb = ((h4 * 0x01020408u) >> 24) & 0xFu;
                const uint32_t yb4 = (uint32_t)(y[0] | (y[1] << 1) | (y[2] << 2) | (y[3] << 3));
                if (chg | (hb ^ yb4)) marks_r |= 1u;
                if (chg) {
                    marks_r |= 256u;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int dy = (int)((yw >> (8 * i)) & 0xFFu) - (int)((yo >> (8 * i)) & 0xFFu);
                        if (dy) du_r += (int64_t)__ldg(L.u + G + i) * dy;
                    }
                    if (lf && (chg & 0xFFu)) marks_r |= 2u;
                    if (rt && (chg >> 24)) marks_r |= 4u;
                    if (tp) marks_r |= 8u;
                    if (bt) marks_r |= 16u;
                    if (zb) marks_r |= 32u;
                    if (zt) marks_r |= 64u;
                }
            };
            {
                const int rr = tid >> 3, cc = (tid & 7) << 2;
                if (zl_) ring_quad(rr, cc, 0);
                if (zh_ && gb.dz > 1) ring_quad(rr, cc, gb.dz - 1);
            }
            {
                const int z = tid >> 3, cc = (tid & 7) << 2;
                const bool zdone = (z == 0 && zl_) || (z == gb.dz - 1 && zh_);
                if (z < gb.dz && !zdone) {
                    if (yl_) ring_quad(0, cc, z);
                    if (yh_) ring_quad(31, cc, z);
                }
            }
#pragma unroll 1
            for (int j = 0; j < 4; ++j) {
                const int rr = tid & 31, z = (tid >> 5) + 8 * j;
                const bool done = (z == 0 && zl_) || (z == gb.dz - 1 && zh_) || (rr == 0 && yl_) || (rr == 31 && yh_);
                if (z < gb.dz && !done) {
                    if (sd & 1u) ring_quad(rr, 0, z);
                    if (sd & 2u) ring_quad(rr, 28, z);
                }
            }
            du_r = warp_sum(du_r);
            const int sq_r = (int)__reduce_add_sync(FULLMASK, (unsigned)ss_r);
            const unsigned fm_r = __reduce_or_sync(FULLMASK, marks_r);
            const unsigned gf_r = __reduce_or_sync(FULLMASK, gfresh);
            if (lane == 0) { red_e[warp] = gf_r; red_s[warp] = sq_r; red_u[warp] = du_r; red_f[warp] = fm_r; }
            __syncthreads();
            if (tid == 0) {
                int64_t S = 0, U = 0;
                unsigned Fm = 0, gf = 0;
                for (int w = 0; w < NT / 32; ++w) { gf |= (unsigned)red_e[w]; S += red_s[w]; U += red_u[w]; Fm |= red_f[w]; }
                // clamp memo: recomputed groups take this pass's bits, the others keep theirs
                const unsigned act = active_groups3(sd);
                const unsigned gbits = (gf & act) | (((unsigned)L.pf[k] >> 1) & ~act);
                L.pu[k] = U;
                L.pr[k] = S;
                L.pf[k] = (gbits ? 1 : 0) | (int)(gbits << 1);
                if (Fm & 1u) mark_dirty(L, k);
                if (Fm & 2u) mark_dirty(L, k - 1);
                if (Fm & 4u) mark_dirty(L, k + 1);
                if (Fm & 8u) mark_dirty(L, k - KX);
                if (Fm & 16u) mark_dirty(L, k + KX);
                if ((Fm & 32u) && k - KYX >= 0) mark_dirty(L, k - KYX);
                if ((Fm & 64u) && k + KYX < L.K) mark_dirty(L, k + KYX);
                ybuf_stamp(L, out)[k] = ep;
                pe_stamp(L)[k] = ep;
                if (Fm & 256u) ychg_stamp(L)[k] = ep;
                agg.add_block(L.pe[k], U, S, gbits ? 1 : 0);
            }
            __syncthreads();
            continue;
        }
        const bool top = r == 0 && up_r, bot = r == 31 && dn_r;
        const bool lft = c0 == 0 && lf_c, rgt = c0 == 28 && rt_c;
        const bool ydn = gb.lo_r + r + 1 < H;             // the +y partner exists
        const bool yld = ydn && (lane >> 3) == 3;          // ... and sits in another warp / block
        const bool xnx = gb.lo_c + c0 + 4 < W;             // the +x partner of the quad's last voxel
        int64_t e_acc = 0, du = 0;
        int ss = 0;
        unsigned marks = 0, clamp_or = 0, gcl = 0;
        const int zend = min((slab + 1) * K2P_SLAB, gb.dz);
        for (int z0 = slab * K2P_SLAB; z0 < zend; z0 += ZB) {
            const int zl = min(z0 + ZB, zend) - 1;        // last plane of the batch
            uint32_t yh4[ZB], yo[ZB], nb[ZB], cnt[ZB], yb[ZB];
            uint2 av[ZB];
            int yr[ZB];
            uint32_t yz = 0;
#pragma unroll
            for (int j = 0; j < ZB; ++j) {
                const int z = z0 + j;
                yh4[j] = yo[j] = nb[j] = cnt[j] = yb[j] = 0;
                av[j] = make_uint2(0, 0);
                yr[j] = 0;
                if (z <= zl) {
                    const int64_t G = G0 + z * HW;
                    yh4[j] = __ldcs(reinterpret_cast<const unsigned int *>(L.yhat + G));
                    av[j] = __ldcs(reinterpret_cast<const uint2 *>(a_in + G));
                    yo[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G));
                    if (want_e) {
                        if (yld) yb[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G + W));
                        if (c0 == 28 && xnx) yr[j] = y_in[G + 4];
                        if (z == zl && (gb.lo_z + z + 1 < D || L.gzd))
                            yz = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G + HW));
                    }
                    if (top) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G - W); }
                    if (bot) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G + W); }
                    if (z == 0 && up_z) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G - HW); }
                    if (z == gb.dz - 1 && dn_z) { cnt[j] += 0x01010101u; nb[j] += *reinterpret_cast<const uint32_t *>(L.yhat + G + HW); }
                    if (lft) { cnt[j] += 1u; nb[j] += L.yhat[G - 1]; }
                    if (rgt) { cnt[j] += 1u << 24; nb[j] += (uint32_t)L.yhat[G + 4] << 24; }
                }
            }
#pragma unroll
            for (int j = 0; j < ZB; ++j) {
                const int z = z0 + j;
                const uint32_t nxt = __shfl_down_sync(FULLMASK, yo[j], 1);
                const uint32_t dnv = __shfl_down_sync(FULLMASK, yo[j], 8);
                if (z > zl) continue;   // uniform over the CTA
                const int64_t G = G0 + z * HW;
                if (want_e) {
                    const uint32_t rw = c0 < 28 ? nxt : (xnx ? (uint32_t)yr[j] : (yo[j] >> 24));
                    int qd = __popc(yo[j] ^ __funnelshift_r(yo[j], rw, 8));
                    if (ydn) qd += __popc(yo[j] ^ (yld ? yb[j] : dnv));
                    if (gb.lo_z + z + 1 < D || L.gzd) qd += __popc(yo[j] ^ (z < zl ? yo[j + 1 < ZB ? j + 1 : j] : yz));
                    e_acc += (int64_t)L.lamw * qd;
                }
                // the quad's update on packed bytes / int16 pairs (quad_update, 2D K2)
                const uint32_t h4 = yh4[j];
                uint2 an2;
                uint32_t qc = 0;
                const uint32_t yn = quad_update(h4, av[j], cnt[j], nb[j], q, 4 * q, an2, qc);
                clamp_or |= qc;
                gcl |= (qc > 1u ? 1u : 0u) << quad_group3(lft, rgt, top, bot, z == 0 && up_z, z == gb.dz - 1 && dn_z);
                const uint32_t hb = bits_b01(h4);
                ss += __popc(hb ^ yn);
                const uint32_t yw = bytes_b01(yn) << 1;   // y2 bytes 0/2
                if (a_out) __stcs(reinterpret_cast<uint2 *>(a_out + G), an2);
                __stcg(reinterpret_cast<unsigned int *>(y_out + G), yw);
                const uint32_t chg = yw ^ yo[j];
                if (chg | (hb ^ yn)) marks |= 1u;
                if (chg) {
                    marks |= 256u;
                    const uint32_t yoj = yo[j];
                    int32_t uq[4];
                    if (L.q3) {
                        const int4 uv = __ldg(reinterpret_cast<const int4 *>(L.u + G));
                        uq[0] = uv.x; uq[1] = uv.y; uq[2] = uv.z; uq[3] = uv.w;
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i) uq[i] = __ldg(L.u + G + i);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        du += (int64_t)uq[i] * ((int)((yw >> (8 * i)) & 0xFFu) - (int)((yoj >> (8 * i)) & 0xFFu));
                    if (lft && (chg & 0xFFu)) marks |= 2u;
                    if (rgt && (chg >> 24)) marks |= 4u;
                    if (top) marks |= 8u;
                    if (bot) marks |= 16u;
                    if (z == 0 && up_z) marks |= 32u;
                    if (z == gb.dz - 1 && dn_z) marks |= 64u;
                }
            }
        }
        e_acc = warp_sum(e_acc);
        du = warp_sum(du);
        const int sq = (int)__reduce_add_sync(FULLMASK, (unsigned)ss);
        const unsigned fm = __reduce_or_sync(FULLMASK, marks | (clamp_or > 1u ? 128u : 0u));
        const unsigned gall = __reduce_or_sync(FULLMASK, gcl);
        if (lane == 0) { red_e[warp] = e_acc; red_s[warp] = sq; red_u[warp] = du; red_f[warp] = fm; red_g[warp] = gall; }
        __syncthreads();
        if (tid == 0) {
            int64_t E = 0, S = 0, U = 0;
            unsigned Fm = 0;
            unsigned gb_ = 0;
            for (int w = 0; w < NT / 32; ++w) { E += red_e[w]; S += red_s[w]; U += red_u[w]; Fm |= red_f[w]; gb_ |= red_g[w]; }
            const int nsk = (gb.dz + K2P_SLAB - 1) / K2P_SLAB;   // this block's slabs
            bool last = true;
            if (nsk > 1) {
                // fold into the block's accumulators; the last slab takes the totals
                // and leaves them zeroed for the next pass
                unsigned long long *acc = slab_acc3(L, k);
                if (E) atomicAdd(&acc[0], (unsigned long long)E);
                if (U) atomicAdd(&acc[1], (unsigned long long)U);
                if (S) atomicAdd(&acc[2], (unsigned long long)S);
                if (Fm | gb_) atomicOr(&acc[3], (unsigned long long)Fm | ((unsigned long long)gb_ << 32));
                __threadfence();
                last = atomicAdd(reinterpret_cast<unsigned int *>(&acc[4]), 1u) == (unsigned)nsk - 1u;
                if (last) {
                    __threadfence();
                    E = (int64_t)__ldcg(&acc[0]);
                    U = (int64_t)__ldcg(&acc[1]);
                    S = (int64_t)__ldcg(&acc[2]);
                    const unsigned long long fg = __ldcg(&acc[3]);
                    Fm = (unsigned)fg;
                    gb_ = (unsigned)(fg >> 32);
                    acc[0] = acc[1] = acc[2] = acc[3] = acc[4] = 0ull;
                }
            }
            if (last) {
            L.pe[k] = E;
            L.pu[k] = U;
            L.pr[k] = S;
            L.pf[k] = ((Fm & 128u) ? 1 : 0) | (int)(gb_ << 1);   // bit 0 clamped, bits 1-27 quad-group clamp memos
            const int KX = L.ax.k, KYX = L.ay.k * L.ax.k;
            if (Fm & 1u) mark_dirty(L, k);
            if (Fm & 2u) mark_dirty(L, k - 1);
            if (Fm & 4u) mark_dirty(L, k + 1);
            if (Fm & 8u) mark_dirty(L, k - KX);
            if (Fm & 16u) mark_dirty(L, k + KX);
            if ((Fm & 32u) && k - KYX >= 0) mark_dirty(L, k - KYX);
            if ((Fm & 64u) && k + KYX < L.K) mark_dirty(L, k + KYX);
            ybuf_stamp(L, out)[k] = ep;
            if (want_e) pe_stamp(L)[k] = ep;
            if (Fm & 256u) ychg_stamp(L)[k] = ep;
            agg.add_block(E, U, S, (Fm & 128u) ? 1 : 0);
            }
        }
        __syncthreads();
    }
    if (tid == 0) pass_tail(L, agg, cur, best, out);
}
