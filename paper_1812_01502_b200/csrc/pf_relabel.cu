// pf_relabel.cu -- the relabelled exchange of a cross stage (RelabelArgs in pf_args.h;
// DESIGN.md reading R24; the surplus sketch of PAPER.md:826-850).
//
//   k_rl_count   one CTA per chunk of kRlChunk positions: both shards' draws of the chunk,
//                counts of "own output wants r'" and "r' output wants own"
//   k_rl_scan    one CTA: exclusive offsets of the chunk counts (fixed order) and the totals
//   k_rl_lists   the two ordered lists (warp ballots + the chunk offsets): own[k] = the k-th
//                own position wanting r', par[k] = the source (in this shard) of the k-th
//                r' output wanting this shard
//   k_rl_pack    the surplus this rank sends: x[par[k]] for k in [kmin, |par|)
//   k_rl_apply   every output once, coalesced: an own-shard draw reads it; the k-th output
//                of list own (kidx) reads x[par[k]] (k < kmin, the swapped draw) or the
//                received surplus (k >= kmin)
// Every draw is the Alg. 3 draw of DESIGN.md §3 (word (i & 3) of Philox block (i >> 2, n,
// RESAMPLE<<24 | s), side low iff (r >> b) < P, index r & (M-1)), on GLOBAL positions.
#include "pf_launch.h"

namespace pfk {

constexpr uint32_t kRlThreads = kRlChunk / 4;

// wants[e] for the 4 positions of quad q of shard `sh`: own shard -> wants r'; partner
// shard -> wants this shard.  src[e] = the local source index (group(l) M + index).
__device__ __forceinline__ void rl_quad(const RelabelArgs& a, uint32_t sh, uint64_t q, uint32_t P, bool* want,
                                        uint32_t* src) {
    const uint64_t gpos = (uint64_t)sh * a.Nloc + 4u * q;
    const uint4 blk = rng_block(a.key, (uint32_t)(gpos >> 2), a.n, kDomainResample, a.s);
    const uint32_t r[4] = {blk.x, blk.y, blk.z, blk.w};
    const bool sh_is_low = (sh == a.rank) ? (a.own_is_low != 0u) : (a.own_is_low == 0u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const bool low = (r[e] >> a.b) < P;
        const bool stays = (low == sh_is_low);  // the draw lies in shard sh itself
        want[e] = !stays;                       // own: wants r'; partner: wants this shard
        const uint32_t l = (uint32_t)(4u * q) + (uint32_t)e;
        src[e] = ((l >> a.b) << a.b) | (r[e] & (a.M - 1u));
    }
}

__global__ void __launch_bounds__(kRlThreads) k_rl_count(const __grid_constant__ RelabelArgs a) {
    __shared__ uint32_t red[2][kRlThreads / 32];
    const uint32_t P = __ldg(a.thr);
    const uint64_t q = (uint64_t)blockIdx.x * kRlThreads + threadIdx.x;
    uint32_t co = 0, cp = 0;
    if (4u * q < a.Nloc) {
        bool w[4];
        uint32_t src[4];
        rl_quad(a, a.rank, q, P, w, src);
        co = (uint32_t)w[0] + w[1] + w[2] + w[3];
        rl_quad(a, a.partner, q, P, w, src);
        cp = (uint32_t)w[0] + w[1] + w[2] + w[3];
    }
    for (int o = 16; o > 0; o >>= 1) {
        co += __shfl_xor_sync(0xffffffffu, co, o);
        cp += __shfl_xor_sync(0xffffffffu, cp, o);
    }
    if ((threadIdx.x & 31u) == 0u) {
        red[0][threadIdx.x >> 5] = co;
        red[1][threadIdx.x >> 5] = cp;
    }
    __syncthreads();
    if (threadIdx.x < 2u) {
        uint32_t t = 0;
        for (uint32_t w = 0; w < kRlThreads / 32; ++w) t += red[threadIdx.x][w];
        a.cnt[(uint64_t)threadIdx.x * a.nchunks + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) k_rl_scan(const __grid_constant__ RelabelArgs a) {
    // two lists; thread-strided serial sums per segment, then a block scan (fixed order)
    __shared__ uint32_t seg[2][1024];
    const uint32_t nc = a.nchunks, per = (nc + 1023u) / 1024u;
    for (uint32_t li = 0; li < 2; ++li) {
        const uint32_t* c = a.cnt + (uint64_t)li * nc;
        uint32_t* o = a.off + (uint64_t)li * nc;
        const uint32_t c0 = threadIdx.x * per, c1 = min(nc, c0 + per);
        uint32_t t = 0;
        for (uint32_t i = c0; i < c1; ++i) t += c[i];
        seg[li][threadIdx.x] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (uint32_t i = 0; i < 1024u; ++i) {
                const uint32_t v = seg[li][i];
                seg[li][i] = acc;
                acc += v;
            }
            a.off[2ull * nc + li] = acc;  // total
        }
        __syncthreads();
        uint32_t acc = seg[li][threadIdx.x];
        for (uint32_t i = c0; i < c1; ++i) {
            o[i] = acc;
            acc += c[i];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kRlThreads) k_rl_lists(const __grid_constant__ RelabelArgs a) {
    __shared__ uint32_t wsum[2][kRlThreads / 32];
    const uint32_t P = __ldg(a.thr);
    const uint64_t q = (uint64_t)blockIdx.x * kRlThreads + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    bool wo[4] = {false, false, false, false}, wp[4] = {false, false, false, false};
    uint32_t so[4], sp[4];
    if (4u * q < a.Nloc) {
        rl_quad(a, a.rank, q, P, wo, so);
        rl_quad(a, a.partner, q, P, wp, sp);
    }
    const uint32_t no = (uint32_t)wo[0] + wo[1] + wo[2] + wo[3], np = (uint32_t)wp[0] + wp[1] + wp[2] + wp[3];
    // inclusive warp scans of the per-thread counts
    uint32_t io = no, ip = np;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t to = __shfl_up_sync(0xffffffffu, io, o), tp = __shfl_up_sync(0xffffffffu, ip, o);
        if (lane >= (uint32_t)o) {
            io += to;
            ip += tp;
        }
    }
    if (lane == 31u) {
        wsum[0][warp] = io;
        wsum[1][warp] = ip;
    }
    __syncthreads();
    uint32_t bo = a.off[blockIdx.x], bp = a.off[(uint64_t)a.nchunks + blockIdx.x];
    for (uint32_t w = 0; w < warp; ++w) {
        bo += wsum[0][w];
        bp += wsum[1][w];
    }
    uint32_t ko = bo + io - no, kp = bp + ip - np;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (wo[e]) {
            a.own[ko] = (uint32_t)(4u * q) + (uint32_t)e;
            a.kidx[4u * q + e] = ko++;  // the output's rank in list own (k_rl_apply)
        }
        if (wp[e]) a.par[kp++] = sp[e];
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_rl_pack(const __grid_constant__ RelabelArgs a) {
    const T* x = reinterpret_cast<const T*>(a.x);
    T* snd = reinterpret_cast<T*>(a.send);
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < a.nsend; k += (uint64_t)gridDim.x * blockDim.x)
        snd[k] = x[a.par[a.kmin + k]];
}

// every output of this shard in one pass, written once and coalesced (4 consecutive
// outputs per thread): a draw inside the shard reads its source; an output of list own
// reads the swapped draw's source (rank k < kmin) or the received surplus (k >= kmin)
template <typename T, bool DBG>
__global__ void __launch_bounds__(256) k_rl_apply(const __grid_constant__ RelabelArgs a) {
    const T* x = reinterpret_cast<const T*>(a.x);
    const T* rcv = reinterpret_cast<const T*>(a.recv);
    T* out = reinterpret_cast<T*>(a.out);
    const uint32_t P = __ldg(a.thr);
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; 4u * q < a.Nloc; q += (uint64_t)gridDim.x * blockDim.x) {
        bool w[4];
        uint32_t src[4];
        rl_quad(a, a.rank, q, P, w, src);
        Vec4<T> v;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t l = (uint32_t)(4u * q) + (uint32_t)e;
            int64_t g;  // global source (debug)
            if (!w[e]) {
                v.v[e] = x[src[e]];
                g = (int64_t)a.rank * (int64_t)a.Nloc + src[e];
            } else {
                const uint32_t k = __ldg(a.kidx + l);
                if (k < a.kmin) {
                    const uint32_t ps = __ldg(a.par + k);
                    v.v[e] = x[ps];
                    g = (int64_t)a.rank * (int64_t)a.Nloc + ps;
                } else {
                    v.v[e] = rcv[k - a.kmin];
                    g = (int64_t)a.partner * (int64_t)a.Nloc + src[e];
                }
            }
            if constexpr (DBG) a.dbg_anc[l] = (int32_t)g;
        }
        if (a.M >= 4u) {
            *reinterpret_cast<Vec4<T>*>(out + 4u * q) = v;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) out[4u * q + e] = v.v[e];
        }
    }
}

void launch_relabel_plan(cudaStream_t st, const RelabelArgs& a) {
    k_rl_count<<<a.nchunks, kRlThreads, 0, st>>>(a);
    k_rl_scan<<<1, 1024, 0, st>>>(a);
}

void launch_relabel_lists(cudaStream_t st, const RelabelArgs& a) { k_rl_lists<<<a.nchunks, kRlThreads, 0, st>>>(a); }

template <typename T>
static void rl_pack_apply(cudaStream_t st, const RelabelArgs& a, bool pack, uint64_t nown, bool dbg) {
    const uint32_t g = 148u * 8u;
    if (pack) {
        if (a.nsend) k_rl_pack<T><<<g, 256, 0, st>>>(a);
        return;
    }
    (void)nown;
    if (dbg) k_rl_apply<T, true><<<g, 256, 0, st>>>(a);
    else k_rl_apply<T, false><<<g, 256, 0, st>>>(a);
}

void launch_relabel_move(cudaStream_t st, int D, const RelabelArgs& a, bool pack, uint64_t nown, bool dbg) {
    switch (D) {
        case 1: rl_pack_apply<float>(st, a, pack, nown, dbg); break;
        case 2: rl_pack_apply<float2>(st, a, pack, nown, dbg); break;
        case 4: rl_pack_apply<float4>(st, a, pack, nown, dbg); break;
        default: rl_pack_apply<State8>(st, a, pack, nown, dbg); break;
    }
}

}  // namespace pfk
