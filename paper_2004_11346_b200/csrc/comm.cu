// Order-sharded SHT over NCCL, entirely behind the C ABI.
//
// Sharding: the independent unit is the order |m| — its plan
// serves +m and -m only (pkg/src/bfsht/sht.py:146,165) — and every
// colatitude row's phi DFT needs every order (sht.py:148,161).  So each rank
// applies the ALT of its own orders (greedy LPT on 2N-|m|), and each
// direction has exactly one exchange: the node halves move between the
// m-major ALT layout (owner of m) and the theta-major DFT layout (owner of
// row pairs r: rows n+r and n-1-r, contiguous row ranges per rank).
//
// The exchange is grouped ncclSend / ncclRecv over NVLink / NVSwitch, one
// message per rank pair.  The forward needs no gather: the ALT's final
// stage writes the row-major node array Yr[r][order][parity] (format.h), so
// the entries destined to rank q — its rows [a_q, b_q) — are already one
// contiguous run of the arena and are sent from there.  The receiver keeps
// the sources' runs back to back; `recv_layout` tells the DFT kernels where
// entry (m, parity, r) sits.  The inverse sends the same runs back into the
// Yr region, and one kernel moves each entry to the m-major node half the
// inverse ALT reads.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, reusing the copy the
// process already has — e.g. the one torch loaded — so one process never
// mixes two NCCL builds); libbfsht_b200.so itself does not link NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bfsht_b200.h"
#include "engine.cuh"

int bf_synth_rows(bfsht_plan *pl, const bf_half *halves, const double *ybuf, int r_begin,
                  int r_count, double *grid, cudaStream_t st);
int bf_anal_rows(bfsht_plan *pl, const bf_half *halves, double *ubuf, int r_begin, int r_count,
                 const double *grid, const double *weights, cudaStream_t st);
int bf_shard_pack(bfsht_plan *pl, const int64_t *off, const double *coeffs, cudaStream_t st);
int bf_shard_unpack(bfsht_plan *pl, const int64_t *off, double *coeffs, cudaStream_t st);

namespace {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
    ncclResult_t (*getVersion)(int *) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

int load_nccl() {
    std::lock_guard<std::mutex> lock(g_nccl_mu);
    if (g_nccl.h) return 0;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        bfsht_set_error(std::string("cannot load NCCL (libnccl.so.2): ") + dlerror());
        return -5;
    }
    NcclApi a;
    a.h = h;
#define BF_SYM(field, name)                                                  \
    a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));           \
    if (!a.field) {                                                           \
        bfsht_set_error(std::string("NCCL symbol missing: ") + name);         \
        return -5;                                                            \
    }
    BF_SYM(getUniqueId, "ncclGetUniqueId");
    BF_SYM(commInitRank, "ncclCommInitRank");
    BF_SYM(commDestroy, "ncclCommDestroy");
    BF_SYM(groupStart, "ncclGroupStart");
    BF_SYM(groupEnd, "ncclGroupEnd");
    BF_SYM(send, "ncclSend");
    BF_SYM(recv, "ncclRecv");
    BF_SYM(errorString, "ncclGetErrorString");
    BF_SYM(getVersion, "ncclGetVersion");
#undef BF_SYM
    g_nccl = a;
    return 0;
}

#define BF_NCCL(call)                                                          \
    do {                                                                       \
        ncclResult_t _r = (call);                                              \
        if (_r != ncclSuccess) {                                               \
            bfsht_set_error(std::string(#call) + ": " + g_nccl.errorString(_r)); \
            return -6;                                                         \
        }                                                                      \
    } while (0)

// columns of the (m, parity) half, 0 when absent (alt.py:102-107)
int half_cols(int n, int m, int par) {
    const int half = par == 0 ? (m + 1) / 2 : m / 2;
    return std::max(n - half, 0);
}

// Inverse: the Yr-ordered entries (row r, half h of this rank) back to the
// m-major node halves the inverse ALT reads (halves[h].y + r).
__global__ void yr_to_halves_kernel(double4 *__restrict__ arena, int64_t yr, int w, int n,
                                    const bf_half *__restrict__ halves) {
    const int64_t total = (int64_t)n * w;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / w), h = (int)(e - (int64_t)r * w);
        const bf_half hf = halves[h];
        if (hf.ncols > 0) arena[(int64_t)hf.y + r] = arena[yr + e];
    }
}

}  // namespace

struct bfsht_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, device = 0;
};

struct bfsht_sharded {
    bfsht_plan *pl = nullptr;
    bfsht_comm *comm = nullptr;
    int n = 0, rank = 0, world = 1;
    int r0 = 0, rc = 0;                   // this rank's row pairs [r0, r0 + rc)
    std::vector<int64_t> send_counts, recv_counts;   // entries per peer
    std::vector<int64_t> send_off, recv_off;         // entry offsets per peer
    bf_half *recv_layout = nullptr;       // device, 4n halves
    double *recvbuf = nullptr;            // device, recv entries x 4 doubles
    int64_t *coeff_off = nullptr;         // device, per plan order (+m then -m)
    int64_t coeff_len = 0;
};

extern "C" {

int bfsht_shard_orders(int n, int nranks, int rank, int32_t *orders, int32_t *count) {
    if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks || !count) {
        bfsht_set_error("bad shard arguments");
        return -1;
    }
    // greedy LPT over m = 0 .. 2N-1 (descending cost 2N - m), ties to the
    // lowest rank: dist.lpt_orders
    std::vector<double> load(nranks, 0.0);
    int32_t c = 0;
    for (int m = 0; m < 2 * n; ++m) {
        int best = 0;
        for (int r = 1; r < nranks; ++r)
            if (load[r] < load[best]) best = r;
        load[best] += 2 * n - m;
        if (best == rank) {
            if (orders) orders[c] = m;
            ++c;
        }
    }
    *count = c;
    return 0;
}

int bfsht_exchange_layout(int n, int nranks, int rank, void *recv_layout, int64_t *send_counts,
                          int64_t *recv_counts) {
    if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks) {
        bfsht_set_error("bad exchange arguments");
        return -1;
    }
    std::vector<std::vector<int32_t>> all(nranks);
    for (int s = 0; s < nranks; ++s) {
        int32_t c = 0;
        all[s].resize(2 * n);
        bfsht_shard_orders(n, nranks, s, all[s].data(), &c);
        all[s].resize(c);
    }
    auto rows = [&](int q) { return std::make_pair((int64_t)q * n / nranks, (int64_t)(q + 1) * n / nranks); };
    const int64_t w = 2 * (int64_t)all[rank].size();
    const int64_t rc = rows(rank).second - rows(rank).first;
    bf_half *lay = static_cast<bf_half *>(recv_layout);
    if (lay) std::memset(lay, 0, sizeof(bf_half) * 4 * (size_t)n);
    int64_t pos = 0;
    for (int s = 0; s < nranks; ++s) {
        const int64_t ws = 2 * (int64_t)all[s].size();
        if (lay)
            for (size_t i = 0; i < all[s].size(); ++i)
                for (int par = 0; par < 2; ++par) {
                    bf_half &hf = lay[2 * all[s][i] + par];
                    hf.m = all[s][i];
                    hf.ncols = half_cols(n, all[s][i], par);
                    hf.x = (int32_t)ws;
                    hf.y = (int32_t)(pos + 2 * (int64_t)i + par);
                }
        if (recv_counts) recv_counts[s] = rc * ws;
        if (send_counts) send_counts[s] = (rows(s).second - rows(s).first) * w;
        pos += rc * ws;
    }
    if (pos > INT32_MAX) {
        bfsht_set_error("exchange layout exceeds int32 entries");
        return -1;
    }
    return 0;
}

int bfsht_comm_unique_id(void *id) {
    if (!id) {
        bfsht_set_error("null id buffer");
        return -1;
    }
    int rc = load_nccl();
    if (rc) return rc;
    ncclUniqueId u;
    BF_NCCL(g_nccl.getUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
    return 0;
}

int bfsht_comm_init(const void *id, int rank, int nranks, bfsht_comm **out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) {
        bfsht_set_error("bad communicator arguments");
        return -1;
    }
    int rc = load_nccl();
    if (rc) return rc;
    auto *c = new bfsht_comm();
    c->rank = rank;
    c->nranks = nranks;
    if (cudaGetDevice(&c->device) != cudaSuccess) {
        delete c;
        bfsht_set_error("no current CUDA device");
        return -2;
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    const ncclResult_t r = g_nccl.commInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
        bfsht_set_error(std::string("ncclCommInitRank: ") + g_nccl.errorString(r));
        delete c;
        return -6;
    }
    *out = c;
    return 0;
}

void bfsht_comm_free(bfsht_comm *c) {
    if (!c) return;
    if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
    delete c;
}

int bfsht_alltoall_transpose(bfsht_comm *c, const double *send, const int64_t *send_counts,
                             double *recv, const int64_t *recv_counts, int64_t entry_doubles,
                             void *stream) {
    if (!c || !send_counts || !recv_counts || entry_doubles < 1) {
        bfsht_set_error("bad all-to-all arguments");
        return -1;
    }
    const cudaStream_t st = (cudaStream_t)stream;
    int64_t so = 0, ro = 0;
    BF_NCCL(g_nccl.groupStart());
    for (int q = 0; q < c->nranks; ++q) {
        if (send_counts[q] > 0)
            BF_NCCL(g_nccl.send(send + so * entry_doubles, (size_t)(send_counts[q] * entry_doubles),
                                ncclFloat64, q, c->comm, st));
        if (recv_counts[q] > 0)
            BF_NCCL(g_nccl.recv(recv + ro * entry_doubles, (size_t)(recv_counts[q] * entry_doubles),
                                ncclFloat64, q, c->comm, st));
        so += send_counts[q];
        ro += recv_counts[q];
    }
    BF_NCCL(g_nccl.groupEnd());
    return 0;
}

int bfsht_sharded_create(bfsht_plan *pl, bfsht_comm *comm, bfsht_sharded **out) {
    if (!pl || !comm || !out) {
        bfsht_set_error("null argument");
        return -1;
    }
    DeviceGuard guard(pl);
    const int n = pl->n, world = comm->nranks, rank = comm->rank;
    std::vector<int32_t> mine(2 * n);
    int32_t cnt = 0;
    bfsht_shard_orders(n, world, rank, mine.data(), &cnt);
    mine.resize(cnt);
    if (mine != pl->orders) {
        bfsht_set_error("plan orders are not this rank's LPT shard (bfsht_shard_orders)");
        return -1;
    }
    auto *s = new bfsht_sharded();
    s->pl = pl;
    s->comm = comm;
    s->n = n;
    s->rank = rank;
    s->world = world;
    s->r0 = (int)((int64_t)rank * n / world);
    s->rc = (int)((int64_t)(rank + 1) * n / world) - s->r0;
    s->send_counts.resize(world);
    s->recv_counts.resize(world);
    std::vector<bf_half> lay(4 * (size_t)n);
    int rc = bfsht_exchange_layout(n, world, rank, lay.data(), s->send_counts.data(),
                                   s->recv_counts.data());
    if (rc) {
        delete s;
        return rc;
    }
    int64_t recv_total = 0;
    for (int64_t v : s->recv_counts) recv_total += v;
    std::vector<int64_t> off(pl->norders + 1, 0);
    for (int o = 0; o < pl->norders; ++o) {
        const int m = pl->orders[o];
        off[o + 1] = off[o] + (2 * (int64_t)n - m) * (m ? 2 : 1);
    }
    s->coeff_len = off[pl->norders];
    auto fail = [&](const char *what) {
        bfsht_set_error(what);
        bfsht_sharded_free(s);
        return -2;
    };
    if (cudaMalloc(&s->recv_layout, sizeof(bf_half) * lay.size()) != cudaSuccess ||
        cudaMemcpy(s->recv_layout, lay.data(), sizeof(bf_half) * lay.size(),
                   cudaMemcpyHostToDevice) != cudaSuccess)
        return fail("exchange layout upload failed");
    if (cudaMalloc(&s->recvbuf, (size_t)std::max<int64_t>(recv_total, 1) * BF_NRHS * 8) != cudaSuccess ||
        cudaMemset(s->recvbuf, 0, (size_t)std::max<int64_t>(recv_total, 1) * BF_NRHS * 8) != cudaSuccess)
        return fail("exchange buffer allocation failed");
    if (cudaMalloc(&s->coeff_off, sizeof(int64_t) * off.size()) != cudaSuccess ||
        cudaMemcpy(s->coeff_off, off.data(), sizeof(int64_t) * off.size(),
                   cudaMemcpyHostToDevice) != cudaSuccess)
        return fail("coefficient offsets upload failed");
    *out = s;
    return 0;
}

void bfsht_sharded_free(bfsht_sharded *s) {
    if (!s) return;
    DeviceGuard guard(s->pl);
    for (void *p : {(void *)s->recv_layout, (void *)s->recvbuf, (void *)s->coeff_off})
        if (p) cudaFree(p);
    delete s;
}

int64_t bfsht_sharded_info(const bfsht_sharded *s, int64_t info[4]) {
    if (!s || !info) return -1;
    info[0] = s->r0;
    info[1] = s->rc;
    info[2] = s->coeff_len;
    int64_t t = 0;
    for (int64_t v : s->recv_counts) t += v;
    info[3] = t;
    return 0;
}

int bfsht_sharded_forward(bfsht_sharded *s, const double *coeffs, double *grid, void *stream) {
    if (!s || !coeffs || !grid) {
        bfsht_set_error("null argument");
        return -1;
    }
    bfsht_plan *pl = s->pl;
    DeviceGuard guard(pl);
    const cudaStream_t st = (cudaStream_t)stream;
    int rc = bf_shard_pack(pl, s->coeff_off, coeffs, st);
    if (rc) return rc;
    rc = bf_alt_apply(pl, BFSHT_FORWARD, st);
    if (rc) return rc;
    // Yr rows of peer q are contiguous: send straight from the arena
    const double *yr = pl->arena + pl->info[10] * BF_NRHS;
    rc = bfsht_alltoall_transpose(s->comm, yr, s->send_counts.data(), s->recvbuf,
                                  s->recv_counts.data(), BF_NRHS, stream);
    if (rc) return rc;
    return bf_synth_rows(pl, s->recv_layout, s->recvbuf, s->r0, s->rc, grid, st);
}

int bfsht_sharded_inverse(bfsht_sharded *s, const double *grid, double *coeffs,
                          const double *weights, void *stream) {
    if (!s || !coeffs || !grid || !weights) {
        bfsht_set_error("null argument");
        return -1;
    }
    bfsht_plan *pl = s->pl;
    DeviceGuard guard(pl);
    const cudaStream_t st = (cudaStream_t)stream;
    int rc = bf_anal_rows(pl, s->recv_layout, s->recvbuf, s->r0, s->rc, grid, weights, st);
    if (rc) return rc;
    double *yr = pl->arena + pl->info[10] * BF_NRHS;
    rc = bfsht_alltoall_transpose(s->comm, s->recvbuf, s->recv_counts.data(), yr,
                                  s->send_counts.data(), BF_NRHS, stream);
    if (rc) return rc;
    const int w = 2 * pl->norders;
    const int64_t total = (int64_t)pl->n * w;
    if (total > 0) {
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)pl->sm_count * 16);
        yr_to_halves_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<double4 *>(pl->arena),
                                                    pl->info[10], w, pl->n, pl->halves);
        BF_CUDA(cudaGetLastError());
        pl->launches += 1;
    }
    rc = bf_alt_apply(pl, BFSHT_INVERSE, st);
    if (rc) return rc;
    return bf_shard_unpack(pl, s->coeff_off, coeffs, st);
}

}  // extern "C"
