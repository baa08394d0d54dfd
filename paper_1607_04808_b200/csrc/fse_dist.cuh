// fse_dist.cuh -- the z-slab (x-plane) decomposition of fse::total_sum with
// PARTITIONED particles and halo exchange.  Included at the end
// of fse_capi.cu: it drives that file's internal stages (prep_points,
// slab_forward_impl, slab_scale_impl, real_part, the quadrature) on each rank's
// local particle set.  Ownership and halo rules: fse_dist_rules.h.
//
// One evaluation, per rank r (G ranks, one GPU each), in lockstep steps with
// one exchange after each:
//   classify   owned sources / targets -> destination ranks (bit masks),
//              per-destination counts                     X0: counts (G x 2 ints)
//   pack       per destination d: the owned sources d needs (spread supports
//              crossing into d's planes, real-space neighbours within rc of
//              d's owned targets) and the owned targets whose support meets
//              d's planes; local arrays = [owned | received, by source rank]
//                                                         X1: ghost particles
//   forward    spread of the local sources onto this slab's planes, z and y
//              FFT passes -> spectrum blocks by ky owner   X2: all-to-all
//   scale      x-FFT, multiplier, inverse x-FFT of this rank's ky rows
//                                                         X3: all-to-all back
//   inverse    inverse y / z passes, this slab's share of the quadrature of
//              every local target (owned and ghost); real-space sum of the
//              owned targets over the local sources (cell geometry of the
//              GLOBAL N, so the bins are the reference's)   X4: ghost partials
//                                                              back to owners
//   finish     u(owned) = own partial + returned partials (ascending source
//              rank) + real space (+ stokeslet self term)
// Exchanges are lists of (peer, pointer, bytes) sends and receives: NCCL
// grouped ncclSend / ncclRecv across GPUs, or a loopback that copies between
// virtual ranks of one process on one device (tests).  No all-reduce: each
// rank returns only its owned targets' velocities.
#pragma once

#include <nccl.h>

#include <functional>
#include <memory>
#include <thread>

#include "fse_dist_rules.h"

namespace fsecu {

#define FSE_NCCL(x)                                                                  \
    do {                                                                             \
        ncclResult_t r_ = (x);                                                       \
        if (r_ != ncclSuccess)                                                       \
            throw Error(FSE_ENCCL, std::string("NCCL error in " #x ": ") +          \
                                       ncclGetErrorString(r_));                      \
    } while (0)

namespace dist {

using fsedist::Geom;

// ---------------------------------------------------------------- kernels
__global__ void k_masks(const double* __restrict__ pos, int64_t n, Geom q, int targets,
                        uint32_t* __restrict__ mask) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double x = pos[3 * i];
    mask[i] = targets ? fsedist::target_mask(x, q) : fsedist::source_mask(x, q);
}

// all destinations at once: segment d of flag (n + 1 entries, the last 0) is
// bit d of the masks, except the own rank's segment (all 0); one scan over the
// G segments then gives every destination's offsets (relative to its
// segment's first offset)
__global__ void k_flag_bits(const uint32_t* __restrict__ mask, int64_t n, int G, int self,
                            int32_t* __restrict__ flag) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= static_cast<int64_t>(G) * (n + 1)) return;
    const int d = static_cast<int>(e / (n + 1));
    const int64_t i = e - static_cast<int64_t>(d) * (n + 1);
    flag[e] = (i < n && d != self) ? static_cast<int32_t>((mask[i] >> d) & 1u) : 0;
}

// cnt[d] = points flagged for destination d (from the scanned segments)
__global__ void k_seg_totals(const int32_t* __restrict__ off, int64_t n, int G,
                             int64_t* __restrict__ cnt) {
    const int d = threadIdx.x;
    if (d < G) cnt[d] = off[static_cast<int64_t>(d) * (n + 1) + n] - off[static_cast<int64_t>(d) * (n + 1)];
}

// idx_d[off - off(segment start)] = i for the flagged points of segment d
__global__ void k_compact_seg(const int32_t* __restrict__ flag, const int32_t* __restrict__ off,
                              int64_t n, int32_t* __restrict__ idx) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n && flag[i]) idx[off[i] - off[0]] = static_cast<int32_t>(i);
}

// out[j * w + c] = in[idx[j] * w + c]
__global__ void k_gather_rows(const double* __restrict__ in, const int32_t* __restrict__ idx,
                              int64_t m, int w, double* __restrict__ out) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= m * w) return;
    const int64_t j = e / w;
    const int c = static_cast<int>(e - j * w);
    out[e] = in[static_cast<int64_t>(idx[j]) * w + c];
}

// u[idx[j] * 3 + c] += add[j * 3 + c]  (idx unique within one call)
__global__ void k_scatter_add3(const double* __restrict__ add, const int32_t* __restrict__ idx,
                               int64_t m, double* __restrict__ u) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= 3 * m) return;
    const int64_t j = e / 3;
    const int c = static_cast<int>(e - 3 * j);
    u[static_cast<int64_t>(idx[j]) * 3 + c] += add[e];
}

inline unsigned nblk(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

// ---------------------------------------------------------------- messages
struct Msg {
    int peer;
    void* ptr;
    size_t bytes;
};
struct Step {
    std::vector<Msg> sends, recvs;
};

// growable device buffer owned by one rank
struct GBuf {
    void* p = nullptr;
    size_t bytes = 0;
    GBuf() = default;
    GBuf(const GBuf&) = delete;
    GBuf& operator=(const GBuf&) = delete;
    ~GBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* get(size_t count) {
        const size_t need = std::max<size_t>(count, 1) * sizeof(T);
        if (need > bytes) {
            if (p) FSE_CU(cudaFree(p));
            p = nullptr;
            bytes = 0;
            FSE_CU(cudaMalloc(&p, need + need / 8));
            bytes = need + need / 8;
        }
        return static_cast<T*>(p);
    }
    template <class T>
    T* ptr() const {
        return static_cast<T*>(p);
    }
};

// ---------------------------------------------------------------- one rank
struct Rank {
    fse_cuda_ctx* c;
    int r, G;
    fse_config cfg{};
    int kind = 0, a = 3;
    GridParams g{};
    Geom q{};
    // inputs (device, caller-owned): owned sources / targets
    const double *pos = nullptr, *str = nullptr, *tgt = nullptr;
    int64_t n_own = 0, nt_own = 0, n_total = 0;
    bool tas = false;
    // classification
    GBuf smask, tmask, flag, off;
    std::vector<std::unique_ptr<GBuf>> sidx, tidx;  // per destination: owned indices
    GBuf cnt_dev;          // [G] source counts, [G] target counts (to each destination)
    GBuf cnt_all;          // G x 2G gathered counts (row s = rank s's counts)
    std::vector<int64_t> scnt, tcnt, rs, rt;  // sent to d / received from s
    // local arrays: [owned | ghosts from rank 0 | 1 | ...]
    GBuf lpos, lstr, ltgt, sendbuf_s, sendbuf_t;
    std::vector<int64_t> soff_send, toff_send;  // offsets (rows) into the send buffers
    int64_t n_loc = 0, nt_loc = 0;
    // spectrum
    GBuf spec_a, spec_b;
    int64_t block = 0;
    // results
    GBuf u_loc, u_ret, u_real;
    std::vector<int64_t> ret_off;

    Rank(fse_cuda_ctx* ctx, int rank, int nranks) : c(ctx), r(rank), G(nranks) {
        for (int d = 0; d < G; ++d) {
            sidx.emplace_back(new GBuf);
            tidx.emplace_back(new GBuf);
        }
    }

    void setup(const fse_config* cf, int k, const double* p, const double* s, int64_t n,
               int64_t ntot, const double* t, int64_t nt, bool targets_are_sources) {
        cfg = *cf;
        kind = k;
        a = arity_of(k);
        g = slab_params(cf, r, G);
        const GridParams g1 = make_grid_params(*cf);
        q = Geom{G, g.nxs, g1.Mt, g1.P, g1.origin, g1.h, cf->rc / g1.h};
        pos = p;
        str = s;
        n_own = n;
        n_total = ntot;
        tas = targets_are_sources;
        tgt = tas ? p : t;
        nt_own = tas ? n : nt;
        block = slab_block_elems(g, a);
    }

    // step 0: masks and per-destination counts; exchange: all-gather of counts
    Step classify() {
        cudaStream_t s = c->s0;
        uint32_t* sm = smask.get<uint32_t>(n_own);
        uint32_t* tm = tmask.get<uint32_t>(nt_own);
        if (n_own > 0) k_masks<<<nblk(n_own), 256, 0, s>>>(pos, n_own, q, 0, sm);
        if (nt_own > 0) k_masks<<<nblk(nt_own), 256, 0, s>>>(tgt, nt_own, q, 1, tm);
        FSE_LAUNCH_CHECK();
        c->launches += 2;
        int64_t* cnt = cnt_dev.get<int64_t>(2 * G);
        FSE_CU(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * 2 * G, s));
        scnt.assign(G, 0);
        tcnt.assign(G, 0);
        // per pass: one flag kernel over all destinations, one scan, one totals
        // kernel; a single host sync for both passes' counts
        int32_t* fl[2] = {nullptr, nullptr};
        int32_t* of[2] = {nullptr, nullptr};
        const int64_t np[2] = {n_own, nt_own};
        const int64_t tot_len = G * (n_own + 1) + G * (nt_own + 1);
        int32_t* f_all = flag.get<int32_t>(tot_len);
        int32_t* o_all = off.get<int32_t>(tot_len);
        fl[0] = f_all;
        of[0] = o_all;
        fl[1] = f_all + G * (n_own + 1);
        of[1] = o_all + G * (n_own + 1);
        for (int pass = 0; pass < 2; ++pass) {
            const int64_t n = np[pass];
            if (n == 0 || G == 1) continue;
            const uint32_t* m = pass ? tm : sm;
            const int64_t len = static_cast<int64_t>(G) * (n + 1);
            k_flag_bits<<<nblk(len), 256, 0, s>>>(m, n, G, r, fl[pass]);
            exclusive_scan(c, s, "dist", fl[pass], of[pass], len);
            k_seg_totals<<<1, 32 * ((G + 31) / 32), 0, s>>>(of[pass], n, G, cnt + pass * G);
            c->launches += 2;
        }
        FSE_LAUNCH_CHECK();
        std::vector<int64_t> h(2 * G, 0);
        FSE_CU(cudaMemcpyAsync(h.data(), cnt, sizeof(int64_t) * 2 * G, cudaMemcpyDeviceToHost, s));
        FSE_CU(cudaStreamSynchronize(s));
        for (int pass = 0; pass < 2; ++pass) {
            const int64_t n = np[pass];
            for (int d = 0; d < G; ++d) {
                if (d == r || n == 0) continue;
                const int64_t tot = h[pass * G + d];
                GBuf& ib = pass ? *tidx[d] : *sidx[d];
                int32_t* idx = ib.get<int32_t>(tot);
                if (tot > 0) {
                    const int64_t seg = static_cast<int64_t>(d) * (n + 1);
                    k_compact_seg<<<nblk(n), 256, 0, s>>>(fl[pass] + seg, of[pass] + seg, n, idx);
                    ++c->launches;
                }
                (pass ? tcnt : scnt)[d] = tot;
            }
        }
        FSE_LAUNCH_CHECK();
        int64_t* all = cnt_all.get<int64_t>(2 * G * G);
        Step st;
        for (int d = 0; d < G; ++d) {
            st.sends.push_back({d, cnt, sizeof(int64_t) * 2 * G});
            st.recvs.push_back({d, all + 2 * G * d, sizeof(int64_t) * 2 * G});
        }
        return st;
    }

    // step 1: pack and exchange ghost particles into the local arrays
    Step pack() {
        cudaStream_t s = c->s0;
        std::vector<int64_t> all(2 * G * G);
        FSE_CU(cudaMemcpyAsync(all.data(), cnt_all.ptr<int64_t>(), sizeof(int64_t) * 2 * G * G,
                               cudaMemcpyDeviceToHost, s));
        FSE_CU(cudaStreamSynchronize(s));
        rs.assign(G, 0);
        rt.assign(G, 0);
        for (int src = 0; src < G; ++src) {
            rs[src] = all[2 * G * src + r];
            rt[src] = all[2 * G * src + G + r];
        }
        int64_t ns = n_own, nts = nt_own;
        for (int src = 0; src < G; ++src) {
            ns += rs[src];
            nts += rt[src];
        }
        n_loc = ns;
        nt_loc = nts;
        double* lp = lpos.get<double>(3 * ns);
        double* ls = lstr.get<double>(static_cast<size_t>(a) * ns);
        double* lt = ltgt.get<double>(3 * nts);
        if (n_own > 0) {
            FSE_CU(cudaMemcpyAsync(lp, pos, sizeof(double) * 3 * n_own, cudaMemcpyDeviceToDevice, s));
            FSE_CU(cudaMemcpyAsync(ls, str, sizeof(double) * a * n_own, cudaMemcpyDeviceToDevice, s));
        }
        if (nt_own > 0)
            FSE_CU(cudaMemcpyAsync(lt, tgt, sizeof(double) * 3 * nt_own, cudaMemcpyDeviceToDevice, s));
        // send buffers: per destination [pos rows | strength rows], then target rows
        int64_t sp = 0, tp = 0;
        soff_send.assign(G + 1, 0);
        toff_send.assign(G + 1, 0);
        for (int d = 0; d < G; ++d) {
            soff_send[d] = sp;
            toff_send[d] = tp;
            sp += scnt[d];
            tp += tcnt[d];
        }
        soff_send[G] = sp;
        toff_send[G] = tp;
        double* sb = sendbuf_s.get<double>(static_cast<size_t>(3 + a) * sp);
        double* tb = sendbuf_t.get<double>(3 * tp);
        Step st;
        for (int d = 0; d < G; ++d) {
            if (scnt[d] > 0) {
                double* bp = sb + (3 + a) * soff_send[d];
                double* bs = bp + 3 * scnt[d];
                k_gather_rows<<<nblk(3 * scnt[d]), 256, 0, s>>>(pos, sidx[d]->ptr<int32_t>(),
                                                                 scnt[d], 3, bp);
                k_gather_rows<<<nblk(a * scnt[d]), 256, 0, s>>>(str, sidx[d]->ptr<int32_t>(),
                                                                 scnt[d], a, bs);
                c->launches += 2;
                st.sends.push_back({d, bp, sizeof(double) * 3 * scnt[d]});
                st.sends.push_back({d, bs, sizeof(double) * a * scnt[d]});
            }
            if (tcnt[d] > 0) {
                double* bt = tb + 3 * toff_send[d];
                k_gather_rows<<<nblk(3 * tcnt[d]), 256, 0, s>>>(tgt, tidx[d]->ptr<int32_t>(),
                                                                 tcnt[d], 3, bt);
                ++c->launches;
                st.sends.push_back({d, bt, sizeof(double) * 3 * tcnt[d]});
            }
        }
        FSE_LAUNCH_CHECK();
        int64_t ps = n_own, pt = nt_own;
        ret_off.assign(G + 1, 0);
        for (int src = 0; src < G; ++src) {
            if (rs[src] > 0) {
                st.recvs.push_back({src, lp + 3 * ps, sizeof(double) * 3 * rs[src]});
                st.recvs.push_back({src, ls + a * ps, sizeof(double) * a * rs[src]});
            }
            if (rt[src] > 0) st.recvs.push_back({src, lt + 3 * pt, sizeof(double) * 3 * rt[src]});
            ps += rs[src];
            pt += rt[src];
        }
        FSE_CU(cudaStreamSynchronize(s));  // send buffers complete before the exchange
        return st;
    }

    // step 2: spread + z/y passes of the local sources -> spectrum blocks by ky owner
    Step forward() {
        double* sa = spec_a.get<double>(2 * static_cast<size_t>(block) * G);
        double* sbk = spec_b.get<double>(2 * static_cast<size_t>(block) * G);
        slab_forward_impl(c, &cfg, kind, lpos.ptr<double>(), lstr.ptr<double>(), n_loc, r, G, sa,
                          nullptr);
        Step st;
        for (int d = 0; d < G; ++d) {
            st.sends.push_back({d, sa + 2 * block * d, sizeof(double) * 2 * block});
            st.recvs.push_back({d, sbk + 2 * block * d, sizeof(double) * 2 * block});
        }
        return st;
    }

    // step 3: x pass + multiplier of this rank's ky rows; blocks back to the x owners
    Step scale(const fse_green* green) {
        double* sa = spec_a.ptr<double>();
        double* sbk = spec_b.ptr<double>();
        slab_scale_impl(c, &cfg, kind, green, r, G, sbk, nullptr);
        Step st;
        for (int d = 0; d < G; ++d) {
            st.sends.push_back({d, sbk + 2 * block * d, sizeof(double) * 2 * block});
            st.recvs.push_back({d, sa + 2 * block * d, sizeof(double) * 2 * block});
        }
        return st;
    }

    // step 4: inverse passes, quadrature partials of all local targets, real space of
    // the owned targets; ghost partials go back to their owners
    Step inverse() {
        Launch L = L0(c);
        const GridParams& gg = g;
        double* ul = u_loc.get<double>(3 * std::max<int64_t>(nt_loc, 1));
        double* uR = u_real.get<double>(3 * std::max<int64_t>(nt_own, 1));
        FSE_CU(cudaMemsetAsync(c->d_flags, 0, 3 * sizeof(int), c->s0));
        FSE_CU(cudaEventRecord(c->ev[EV_START], c->s0));
        FSE_CU(cudaStreamWaitEvent(c->s1, c->ev[EV_START], 0));
        if (nt_own > 0)
            real_part(c, kind, lpos.ptr<double>(), lstr.ptr<double>(), n_loc, cfg.L, cfg.xi,
                      cfg.rc, ltgt.ptr<double>(), nt_own, false, uR, 0, 1, n_total);
        FSE_CU(cudaEventRecord(c->ev[EV_JOIN], c->s1));
        double* qtab = buf<double>(c, "qtab", gg.P);
        launch_quad_table(L, gg, qtab);
        double* W = buf<double>(c, "R", static_cast<size_t>(a) * gg.comp);
        double2* Bs = buf<double2>(c, "B", static_cast<size_t>(a) * gg.nx * gg.Mt * gg.Dh);
        const FftPlanDev& fp = fft_plan(c, gg.D);
        launch_fft_inverse_yz(L, fp.host, fp.tw, gg, a,
                              reinterpret_cast<double2*>(spec_a.ptr<double>()), Bs, W);
        if (nt_loc > 0) {
            Sorted tg = prep_points(c, gg, "ft_", ltgt.ptr<double>(), nullptr, 0, nt_loc, 1, qtab);
            if (G > 1) FSE_CU(cudaMemsetAsync(ul, 0, sizeof(double) * 3 * nt_loc, c->s0));
            quadrature(c, gg, tg, nt_loc, W, gg.h * gg.h * gg.h, ul, false);
        }
        FSE_CU(cudaStreamWaitEvent(c->s0, c->ev[EV_JOIN], 0));
        raise_flags(c);  // synchronises s0 (partials complete before they are sent)
        Step st;
        int64_t pt = nt_own;
        for (int src = 0; src < G; ++src) {
            if (rt[src] > 0) st.sends.push_back({src, ul + 3 * pt, sizeof(double) * 3 * rt[src]});
            pt += rt[src];
        }
        int64_t tot = 0;
        for (int d = 0; d < G; ++d) tot += tcnt[d];
        double* ret = u_ret.get<double>(3 * std::max<int64_t>(tot, 1));
        int64_t o = 0;
        for (int d = 0; d < G; ++d) {
            ret_off[d] = o;
            if (tcnt[d] > 0) st.recvs.push_back({d, ret + 3 * o, sizeof(double) * 3 * tcnt[d]});
            o += tcnt[d];
        }
        ret_off[G] = o;
        return st;
    }

    // step 5: owned velocities (in the order of the owned target array)
    void finish(double* d_u) {
        Launch L = L0(c);
        double* ul = u_loc.ptr<double>();
        const double* ret = u_ret.ptr<double>();
        for (int d = 0; d < G; ++d)
            if (tcnt[d] > 0) {
                k_scatter_add3<<<nblk(3 * tcnt[d]), 256, 0, c->s0>>>(
                    ret + 3 * ret_off[d], tidx[d]->ptr<int32_t>(), tcnt[d], ul);
                FSE_LAUNCH_CHECK();
                ++c->launches;
            }
        if (nt_own > 0) {
            const bool self = tas && kind == FSE_STOKESLET;
            launch_epilogue(L, nt_own, ul, u_real.ptr<double>(),
                            self ? str : nullptr, self ? -4.0 * cfg.xi / std::sqrt(M_PI) : 0.0,
                            d_u);
        }
        FSE_CU(cudaStreamSynchronize(c->s0));
    }
};

// ---------------------------------------------------------------- exchanges
struct NcclComm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    ~NcclComm() {
        if (comm) ncclCommDestroy(comm);
    }
};

void run_nccl(const NcclComm& nc, cudaStream_t s, int self, const Step& st) {
    // self messages are device copies (in order); the rest one NCCL group
    std::vector<Msg> ss, rr;
    for (const Msg& m : st.sends)
        if (m.peer == self) ss.push_back(m);
    for (const Msg& m : st.recvs)
        if (m.peer == self) rr.push_back(m);
    if (ss.size() != rr.size()) invalid("dist: unmatched self messages");
    for (size_t i = 0; i < ss.size(); ++i)
        if (ss[i].bytes)
            FSE_CU(cudaMemcpyAsync(rr[i].ptr, ss[i].ptr, ss[i].bytes, cudaMemcpyDeviceToDevice, s));
    FSE_NCCL(ncclGroupStart());
    for (const Msg& m : st.sends)
        if (m.peer != self && m.bytes) FSE_NCCL(ncclSend(m.ptr, m.bytes, ncclChar, m.peer, nc.comm, s));
    for (const Msg& m : st.recvs)
        if (m.peer != self && m.bytes) FSE_NCCL(ncclRecv(m.ptr, m.bytes, ncclChar, m.peer, nc.comm, s));
    FSE_NCCL(ncclGroupEnd());
    // stream-ordered: the next step's kernels on s queue behind the transfers;
    // the host only waits where it needs received counts (pack)
}

// virtual ranks of one process on one device: copy every send to the matching
// receive (same (sender, receiver) pair, in order)
void run_loopback(std::vector<Step>& steps, cudaStream_t s) {
    const int G = static_cast<int>(steps.size());
    for (int d = 0; d < G; ++d) {
        std::vector<size_t> used(G, 0);
        for (const Msg& rv : steps[d].recvs) {
            const int src = rv.peer;
            size_t k = 0, seen = 0;
            for (; k < steps[src].sends.size(); ++k)
                if (steps[src].sends[k].peer == d && seen++ == used[src]) break;
            if (k == steps[src].sends.size()) invalid("dist loopback: unmatched receive");
            ++used[src];
            const Msg& sd = steps[src].sends[k];
            if (sd.bytes != rv.bytes) invalid("dist loopback: message size mismatch");
            if (sd.bytes)
                FSE_CU(cudaMemcpyAsync(rv.ptr, sd.ptr, sd.bytes, cudaMemcpyDeviceToDevice, s));
        }
    }
    FSE_CU(cudaStreamSynchronize(s));
}

}  // namespace dist
}  // namespace fsecu

struct fse_dist {
    fse_cuda_ctx* ctx = nullptr;
    fsecu::dist::NcclComm nc;
    std::unique_ptr<fsecu::dist::Rank> rank;
};

struct fse_multi {
    std::vector<int> devices;
    std::vector<fse_cuda_ctx*> ctx;
    std::vector<fsecu::dist::NcclComm> nc;
    std::vector<std::unique_ptr<fsecu::dist::Rank>> ranks;
    std::vector<fse_green*> greens;
    int green_kind = -1, green_Mt = 0;
    double green_Lt = 0, green_sf = 0;
    const double* green_src = nullptr;  // caller's table the device copies came from
    std::vector<std::unique_ptr<fsecu::dist::GBuf>> dp, ds, dt, du;
    std::string err;
    std::mutex mu;
};

namespace {

using namespace fsecu::dist;

void run_rank_steps(Rank& R, const NcclComm& nc, cudaStream_t s, const fse_green* green) {
    const int me = nc.rank;
    run_nccl(nc, s, me, R.classify());
    run_nccl(nc, s, me, R.pack());
    run_nccl(nc, s, me, R.forward());
    run_nccl(nc, s, me, R.scale(green));
    run_nccl(nc, s, me, R.inverse());
}

// the steps of one evaluation on one NCCL rank
void dist_total_sum(fse_dist* D, const fse_config* cfg, int kind, const double* d_pos,
                    const double* d_str, int64_t n_own, int64_t n_total, const double* d_tgt,
                    int64_t nt_own, int tas, const fse_green* green, double* d_u) {
    check_kind(kind);
    check_cfg(cfg);
    check_green(cfg, kind, green);
    if (n_own < 0 || nt_own < 0 || n_total < n_own) invalid("dist: bad point counts");
    fse_cuda_ctx* c = D->ctx;
    Rank& R = *D->rank;
    R.setup(cfg, kind, d_pos, d_str, n_own, n_total, d_tgt, nt_own, tas != 0);
    run_rank_steps(R, D->nc, c->s0, green);
    R.finish(d_u);
}

}  // namespace

extern "C" {

fse_status fse_cuda_nccl_unique_id(void* id128) {
    if (!id128) return FSE_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return FSE_ENCCL;
    std::memcpy(id128, &id, sizeof id);
    return FSE_OK;
}

fse_status fse_cuda_dist_create(fse_cuda_ctx* c, int rank, int nranks, const void* id128,
                                fse_dist** out) {
    return api(c, [&] {
        if (!out || !id128) invalid("null pointer");
        if (nranks < 1 || nranks > kMaxSlabs || rank < 0 || rank >= nranks)
            invalid("dist: need 0 <= rank < nranks <= 16");
        auto D = std::make_unique<fse_dist>();
        D->ctx = c;
        D->nc.rank = rank;
        D->nc.nranks = nranks;
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        FSE_NCCL(ncclCommInitRank(&D->nc.comm, nranks, id, rank));
        D->rank = std::make_unique<Rank>(c, rank, nranks);
        *out = D.release();
    });
}

void fse_cuda_dist_destroy(fse_dist* D) { delete D; }

fse_status fse_cuda_dist_total_sum(fse_dist* D, const fse_config* cfg, int kind,
                                   const double* d_pos, const double* d_str, int64_t n_own,
                                   int64_t n_total, const double* d_tgt, int64_t nt_own, int tas,
                                   const fse_green* green, double* d_u) {
    if (!D) return FSE_EINVAL;
    return api(D->ctx, [&] {
        dist_total_sum(D, cfg, kind, d_pos, d_str, n_own, n_total, d_tgt, nt_own, tas, green, d_u);
    });
}

// G virtual ranks on this context's device, exchanges as device copies: the whole
// partitioned algorithm on one GPU (tests).  Inputs: ALL points (device), which
// are partitioned here by the ownership rule; u in caller order.
fse_status fse_cuda_dist_virtual_total_sum(fse_cuda_ctx* c, int nranks, const fse_config* cfg,
                                           int kind, const double* d_pos, const double* d_str,
                                           int64_t n, const double* d_tgt, int64_t nt, int tas,
                                           const fse_green* green, double* d_u, double* prof) {
    return api(c, [&] {
        check_kind(kind);
        check_cfg(cfg);
        check_green(cfg, kind, green);
        if (nranks < 1 || nranks > kMaxSlabs) invalid("dist: 1 <= nranks <= 16");
        const int G = nranks, a = arity_of(kind);
        const GridParams g0 = slab_params(cfg, 0, G);
        const GridParams g1 = make_grid_params(*cfg);
        const Geom q{G, g0.nxs, g1.Mt, g1.P, g1.origin, g1.h, cfg->rc / g1.h};
        if (tas) d_tgt = d_pos, nt = n;
        // partition on the host by the shared rule (test path)
        std::vector<double> hp(3 * n), hs(static_cast<size_t>(a) * n), ht(3 * nt);
        FSE_CU(cudaMemcpy(hp.data(), d_pos, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
        FSE_CU(cudaMemcpy(hs.data(), d_str, sizeof(double) * a * n, cudaMemcpyDeviceToHost));
        FSE_CU(cudaMemcpy(ht.data(), d_tgt, sizeof(double) * 3 * nt, cudaMemcpyDeviceToHost));
        std::vector<std::vector<int64_t>> own_s(G), own_t(G);
        for (int64_t i = 0; i < n; ++i) own_s[fsedist::owner_of(hp[3 * i], q)].push_back(i);
        for (int64_t i = 0; i < nt; ++i) own_t[fsedist::owner_of(ht[3 * i], q)].push_back(i);
        std::vector<std::unique_ptr<Rank>> ranks;
        std::vector<std::unique_ptr<GBuf>> in_p, in_s, in_t, out_u;
        for (int r = 0; r < G; ++r) {
            ranks.emplace_back(new Rank(c, r, G));
            in_p.emplace_back(new GBuf);
            in_s.emplace_back(new GBuf);
            in_t.emplace_back(new GBuf);
            out_u.emplace_back(new GBuf);
            std::vector<double> bp, bs, bt;
            for (int64_t i : own_s[r]) {
                bp.insert(bp.end(), &hp[3 * i], &hp[3 * i + 3]);
                bs.insert(bs.end(), &hs[a * i], &hs[a * i + a]);
            }
            for (int64_t i : own_t[r]) bt.insert(bt.end(), &ht[3 * i], &ht[3 * i + 3]);
            double* dp = in_p[r]->get<double>(bp.size());
            double* ds = in_s[r]->get<double>(bs.size());
            double* dt = in_t[r]->get<double>(bt.size());
            if (!bp.empty()) h2d(c, dp, bp.data(), sizeof(double) * bp.size());
            if (!bs.empty()) h2d(c, ds, bs.data(), sizeof(double) * bs.size());
            if (!bt.empty()) h2d(c, dt, bt.data(), sizeof(double) * bt.size());
            out_u[r]->get<double>(3 * std::max<size_t>(own_t[r].size(), 1));
            ranks[r]->setup(cfg, kind, dp, ds, static_cast<int64_t>(own_s[r].size()), n, dt,
                            static_cast<int64_t>(own_t[r].size()), tas != 0);
        }
        // prof (optional): per rank and step (classify, pack, forward, scale,
        // inverse, finish) the step's time on the device (ms, the rank running
        // alone) and the bytes it sends to other ranks: [r][step][time, bytes]
        int step_no = 0;
        bool timing = prof != nullptr;
        auto record = [&](int r, int stp, double ms, double bytes) {
            if (timing) {
                prof[(r * 6 + stp) * 2] = ms;
                prof[(r * 6 + stp) * 2 + 1] = bytes;
            }
        };
        auto step_all = [&](const std::function<Step(Rank&)>& f) {
            std::vector<Step> st;
            for (int r = 0; r < G; ++r) {
                FSE_CU(cudaDeviceSynchronize());
                const auto t0 = std::chrono::steady_clock::now();
                st.push_back(f(*ranks[r]));
                FSE_CU(cudaDeviceSynchronize());
                const double ms =
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                        .count();
                double bytes = 0;
                for (const Msg& m : st.back().sends)
                    if (m.peer != r) bytes += static_cast<double>(m.bytes);
                record(r, step_no, ms, bytes);
            }
            run_loopback(st, c->s0);
            ++step_no;
        };
        // with a profile the steps run twice and the second pass is recorded: the
        // first one allocates every rank's buffers (cudaMalloc is synchronous and
        // would otherwise be timed inside the steps)
        for (int pass = prof ? 0 : 1; pass < 2; ++pass) {
            timing = prof != nullptr && pass == 1;
            step_no = 0;
            step_all([](Rank& R) { return R.classify(); });
            step_all([](Rank& R) { return R.pack(); });
            step_all([](Rank& R) { return R.forward(); });
            step_all([&](Rank& R) { return R.scale(green); });
            step_all([](Rank& R) { return R.inverse(); });
            if (pass == 0)
                for (int r = 0; r < G; ++r) ranks[r]->finish(out_u[r]->ptr<double>());
        }
        timing = prof != nullptr;
        std::vector<double> hu(3 * nt);
        for (int r = 0; r < G; ++r) {
            FSE_CU(cudaDeviceSynchronize());
            const auto t0 = std::chrono::steady_clock::now();
            ranks[r]->finish(out_u[r]->ptr<double>());
            record(r, 5,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count(),
                   0.0);
            std::vector<double> ur(3 * own_t[r].size());
            if (!ur.empty()) d2h(c, ur.data(), out_u[r]->ptr<double>(), sizeof(double) * ur.size());
            for (size_t j = 0; j < own_t[r].size(); ++j)
                for (int k = 0; k < 3; ++k) hu[3 * own_t[r][j] + k] = ur[3 * j + k];
        }
        h2d(c, d_u, hu.data(), sizeof(double) * hu.size());
    });
}

// ---- one process, several GPUs (a multi-device context holding the
// NCCL communicators of ncclCommInitAll): host buffers in and out, like
// fse::total_sum; one host thread per device runs that device's rank.
fse_status fse_cuda_multi_create(const int* devices, int ndev, fse_multi** out) {
    if (!out || !devices || ndev < 1 || ndev > kMaxSlabs) return FSE_EINVAL;
    *out = nullptr;
    auto M = std::make_unique<fse_multi>();
    M->devices.assign(devices, devices + ndev);
    for (int r = 0; r < ndev; ++r) {
        fse_cuda_ctx* c = nullptr;
        const fse_status st = fse_cuda_create(devices[r], &c);
        if (st != FSE_OK) {
            for (fse_cuda_ctx* x : M->ctx) fse_cuda_destroy(x);
            return st;
        }
        M->ctx.push_back(c);
    }
    std::vector<ncclComm_t> comms(ndev);
    if (ncclCommInitAll(comms.data(), ndev, devices) != ncclSuccess) {
        for (fse_cuda_ctx* x : M->ctx) fse_cuda_destroy(x);
        return FSE_ENCCL;
    }
    M->nc.resize(ndev);
    for (int r = 0; r < ndev; ++r) {
        M->nc[r].comm = comms[r];
        M->nc[r].rank = r;
        M->nc[r].nranks = ndev;
        M->ranks.emplace_back(new Rank(M->ctx[r], r, ndev));
        M->dp.emplace_back(new GBuf);
        M->ds.emplace_back(new GBuf);
        M->dt.emplace_back(new GBuf);
        M->du.emplace_back(new GBuf);
    }
    M->greens.assign(ndev, nullptr);
    *out = M.release();
    return FSE_OK;
}

void fse_cuda_multi_destroy(fse_multi* M) {
    if (!M) return;
    for (size_t r = 0; r < M->ctx.size(); ++r) {
        cudaSetDevice(M->devices[r]);
        M->ranks[r].reset();
        M->dp[r].reset();
        M->ds[r].reset();
        M->dt[r].reset();
        M->du[r].reset();
        if (M->greens[r]) fse_cuda_green_free(M->greens[r]);
    }
    M->nc.clear();  // ncclCommDestroy
    for (fse_cuda_ctx* c : M->ctx) fse_cuda_destroy(c);
    delete M;
}

const char* fse_cuda_multi_last_error(const fse_multi* M) { return M ? M->err.c_str() : ""; }

fse_status fse_cuda_multi_total_sum(fse_multi* M, const fse_config* cfg, int kind,
                                    const double* pos, const double* str, int64_t n,
                                    double box_side, const double* tgt, int64_t nt, int tas,
                                    const double* green_full, double* u, fse_timings* tm) {
    if (!M) return FSE_EINVAL;
    std::lock_guard<std::mutex> lk(M->mu);
    M->err.clear();
    const auto t_start = std::chrono::steady_clock::now();
    try {
        check_kind(kind);
        check_cfg(cfg);
        if (n < 1 || nt < 0 || !pos || !str || !u || (nt > 0 && !tgt)) invalid("null pointer");
        if (std::abs(box_side - cfg->L) > 1e-12 * cfg->L)
            invalid("spread: config box does not match system");
        const int G = static_cast<int>(M->ctx.size()), a = arity_of(kind);
        const bool same = tas < 0 ? (n == nt && host_equal(pos, tgt, n)) : tas != 0;
        if (same) tgt = pos, nt = n;
        const GridParams g0 = slab_params(cfg, 0, G);
        const GridParams g1 = make_grid_params(*cfg);
        const Geom q{G, g0.nxs, g1.Mt, g1.P, g1.origin, g1.h, cfg->rc / g1.h};
        // host-side checks of the device flags (a rank failing inside the NCCL
        // steps would leave its peers waiting): supports inside the grid
        // (ewald.cpp:87-91) and targets inside the box (ewald.cpp:299-302)
        auto check_points = [&](const double* p, int64_t m, bool box) {
            for (int64_t i = 0; i < 3 * m; ++i) {
                const double x = p[i];
                const int f = fsedist::support_first(fsedist::plane_coord(x, q), q);
                if (!(x == x) || f < 0 || f + g1.P > g1.Mt)
                    invalid("spread/quadrature: point support exceeds grid");
                if (box && !(x >= 0.0 && x <= cfg->L)) invalid("fourier_sum: target outside [0,L]^3");
            }
        };
        check_points(pos, n, false);
        if (!same) check_points(tgt, nt, true);
        // partition by owner
        std::vector<std::vector<int64_t>> own_s(G), own_t(G);
        for (int64_t i = 0; i < n; ++i) own_s[fsedist::owner_of(pos[3 * i], q)].push_back(i);
        if (!same)
            for (int64_t i = 0; i < nt; ++i) own_t[fsedist::owner_of(tgt[3 * i], q)].push_back(i);
        // Green's table on every device: the caller's (D^3 reference layout) or
        // the GPU precompute; cached by kind, geometry and source table
        const int gk = kind == FSE_ROTLET ? FSE_HARMONIC : FSE_BIHARMONIC;
        if (gk != M->green_kind || cfg->Mtilde != M->green_Mt || cfg->Ltilde != M->green_Lt ||
            cfg->sf != M->green_sf || green_full != M->green_src) {
            const int D = 2 * cfg->Mtilde;
            for (int r = 0; r < G; ++r) {
                Guard gd(M->ctx[r]);
                fse_cuda_ctx* c = M->ctx[r];
                if (M->greens[r]) fse_cuda_green_free(M->greens[r]);
                M->greens[r] = nullptr;
                if (green_full) {
                    fse_green* gr = new_green(c, gk, cfg->Ltilde, cfg->Mtilde,
                                              cfg->Ltilde / cfg->Mtilde, std::sqrt(3.0) * cfg->Ltilde);
                    DevScratch scratch;
                    const size_t nfull = static_cast<size_t>(D) * D * D;
                    double* tmp = scratch.alloc<double>(nfull);
                    h2d(c, tmp, green_full, nfull * sizeof(double));
                    launch_green_full_to_half(L0(c), D, tmp, gr->d_half);
                    FSE_CU(cudaStreamSynchronize(c->s0));
                    M->greens[r] = gr;
                } else {
                    M->greens[r] = green_precompute(c, gk, cfg->Ltilde, cfg->Mtilde, cfg->sf);
                }
            }
            M->green_src = green_full;
            M->green_kind = gk;
            M->green_Mt = cfg->Mtilde;
            M->green_Lt = cfg->Ltilde;
            M->green_sf = cfg->sf;
        }
        std::vector<std::string> errs(G);
        std::vector<std::vector<double>> hu(G);
        auto work = [&](int r) {
            try {
                fse_cuda_ctx* c = M->ctx[r];
                Guard gd(c);
                const auto& os = own_s[r];
                const auto& ot = same ? own_s[r] : own_t[r];
                std::vector<double> bp(3 * os.size()), bs(static_cast<size_t>(a) * os.size()),
                    bt(same ? 0 : 3 * ot.size());
                for (size_t j = 0; j < os.size(); ++j) {
                    std::memcpy(&bp[3 * j], pos + 3 * os[j], 3 * sizeof(double));
                    std::memcpy(&bs[a * j], str + a * os[j], a * sizeof(double));
                }
                if (!same)
                    for (size_t j = 0; j < ot.size(); ++j)
                        std::memcpy(&bt[3 * j], tgt + 3 * ot[j], 3 * sizeof(double));
                double* dp = M->dp[r]->get<double>(bp.size());
                double* ds = M->ds[r]->get<double>(bs.size());
                double* dt = same ? dp : M->dt[r]->get<double>(bt.size());
                double* du = M->du[r]->get<double>(3 * std::max<size_t>(ot.size(), 1));
                if (!bp.empty()) h2d(c, dp, bp.data(), sizeof(double) * bp.size());
                if (!bs.empty()) h2d(c, ds, bs.data(), sizeof(double) * bs.size());
                if (!bt.empty()) h2d(c, dt, bt.data(), sizeof(double) * bt.size());
                Rank& R = *M->ranks[r];
                R.setup(cfg, kind, dp, ds, static_cast<int64_t>(os.size()), n, dt,
                        static_cast<int64_t>(ot.size()), same);
                run_rank_steps(R, M->nc[r], c->s0, M->greens[r]);
                R.finish(du);
                hu[r].resize(3 * ot.size());
                if (!hu[r].empty()) d2h(c, hu[r].data(), du, sizeof(double) * hu[r].size());
            } catch (const std::exception& e) {
                errs[r] = e.what();
            }
        };
        std::vector<std::thread> th;
        for (int r = 0; r < G; ++r) th.emplace_back(work, r);
        for (auto& t : th) t.join();
        for (int r = 0; r < G; ++r)
            if (!errs[r].empty()) throw Error(FSE_ERUNTIME, "rank " + std::to_string(r) + ": " + errs[r]);
        for (int r = 0; r < G; ++r) {
            const auto& ot = same ? own_s[r] : own_t[r];
            for (size_t j = 0; j < ot.size(); ++j)
                std::memcpy(u + 3 * ot[j], &hu[r][3 * j], 3 * sizeof(double));
        }
        if (tm)  // only the whole call (host wall clock, transfers included) is timed
            tm->total += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start)
                             .count();
        return FSE_OK;
    } catch (const Error& e) {
        M->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        M->err = e.what();
        return FSE_ERUNTIME;
    }
}

}  // extern "C"
