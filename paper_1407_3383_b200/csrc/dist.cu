// dist.cu -- the distributed transform and integer product behind the C ABI
// (SURVEY §8(b) mm_dist_create / mm_ntt_forward_dist / mm_int_mul_u16_dist,
// §8(e); Algorithm 1 split across ranks).
//
// One process per GPU.  A communicator is built from an NCCL unique id that
// the caller broadcasts (e.g. over torch.distributed); NCCL is not linked:
// libnccl.so.2 is dlopen'ed, which returns the copy torch already loaded into
// the process (RTLD_NOLOAD first), so the library and torch share one NCCL.
//
// Layouts (rank g of G; the plan's n = n2 x n1, c1 = n1 / G, r2 = n2 / G):
//   forward input  : [n2][c1] column block = natural columns [g c1, (g+1) c1)
//   forward output : [r2][n1] row block = bit-mirrored positions [g r2 n1, (g+1) r2 n1)
//   inverse        : the reverse (row block in, column block out, n^-1 applied)
// Steps 1-2 (column TFFTs + twiddle) run on the column block, one all-to-all
// moves row block h of every column block to rank h ("the matrix
// transposition"), steps 3-4 run on the received segments in place.
//
// Transport: NCCL grouped send/recv (default), or -- after mm_dist_p2p_enable
// -- the fused column pass that stores its rows straight into the peers'
// receive buffers over NVLink (CUDA IPC, mm_ntt_fwd_cols_p2p), ordered by
// device-side flags instead of a host barrier: after its column pass a rank
// raises ready[g] = epoch in every peer's flag page (system-scope release),
// the row pass starts once all G ready flags reach the epoch (acquire), and
// after its row pass a rank raises free[g] = epoch, which a peer waits for
// before it writes the same receive buffer again two epochs later (the
// receive buffers alternate by epoch parity).  Everything is stream-ordered
// on the caller's stream; no host synchronisation in the compute calls.
#include "common.h"
#include <dlfcn.h>
#include <nccl.h>
#include <map>
#include <mutex>
#include <new>
#include <string.h>

namespace mm {

// ---------------------------------------------------------------- NCCL entry points (dlopen)
struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*);
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*commDestroy)(ncclComm_t);
    ncclResult_t (*groupStart)();
    ncclResult_t (*groupEnd)();
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    const char* (*errorString)(ncclResult_t);
    ncclResult_t (*getVersion)(int*);
    bool ok = false;
};

static NcclApi* nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy torch loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
#define MM_SYM(field, name) api.field = (decltype(api.field))dlsym(h, name)
        MM_SYM(getUniqueId, "ncclGetUniqueId");
        MM_SYM(commInitRank, "ncclCommInitRank");
        MM_SYM(commDestroy, "ncclCommDestroy");
        MM_SYM(groupStart, "ncclGroupStart");
        MM_SYM(groupEnd, "ncclGroupEnd");
        MM_SYM(send, "ncclSend");
        MM_SYM(recv, "ncclRecv");
        MM_SYM(allGather, "ncclAllGather");
        MM_SYM(errorString, "ncclGetErrorString");
        MM_SYM(getVersion, "ncclGetVersion");
#undef MM_SYM
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.groupStart && api.groupEnd && api.send &&
                 api.recv && api.allGather && api.errorString;
    });
    return api.ok ? &api : nullptr;
}

#define MM_NCCL_TRY(call)                                                                            \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess) return set_err(MM_E_NCCL, "%s failed: %s", #call, N->errorString(r_)); \
    } while (0)

// ---------------------------------------------------------------- device-side flags
struct PeerFlags {
    unsigned long long* p[8];
};
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* a, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
// thread h raises slot `slot` of peer h's flag page to v (after a system-scope
// fence, so the stores of the preceding kernel on this stream are ordered first)
__global__ void k_dist_signal(PeerFlags peers, int G, int slot, unsigned long long v) {
    const int h = threadIdx.x;
    if (h < G) {
        __threadfence_system();
        st_release_sys(peers.p[h] + slot, v);
    }
}
// wait until flags[base + h] >= target for every h < G; gives up after ~20 s
// (a dead peer), recording the slot in *err instead of hanging the device
__global__ void k_dist_wait(const unsigned long long* flags, int base, int G, unsigned long long target,
                            unsigned long long* err) {
    const int h = threadIdx.x;
    if (h < G) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (ld_acquire_sys(flags + base + h) < target) {
            __nanosleep(256);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 20000000000ull) {
                atomicExch(err, 1ull + (unsigned long long)(base + h));
                break;
            }
        }
    }
    __syncthreads();
}

}  // namespace mm

using namespace mm;

struct mm_dist {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, dev = 0;
    // peer-memory transport
    bool p2p = false;
    size_t p2p_bytes = 0;            // per receive buffer
    char* base = nullptr;            // [recv0 | recv1 | flag page] (one cudaMalloc, IPC-exported)
    void* peer_recv[2][8] = {};
    PeerFlags peer_flags{};          // flag pages of every rank (own = local)
    char* peer_base[8] = {};         // opened IPC bases (nullptr for self)
    unsigned long long epoch = 0;
    std::mutex mu;
    std::map<int, mm_ntt_plan*> plans;   // Goldilocks plans for the integer product
};

namespace mm {
static size_t flag_page_bytes(int G) { return 2 * 8 * (size_t)G + 8 + 512; }   // ready[G], free[G], error word (padded)
}

extern "C" mm_status mm_dist_unique_id(void* id_out) {
    if (!id_out) return set_err(MM_E_ARG, "null argument");
    NcclApi* N = nccl();
    if (!N) return set_err(MM_E_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    MM_NCCL_TRY(N->getUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return MM_OK;
}

extern "C" mm_status mm_dist_create(const void* nccl_unique_id, int rank, int world, mm_dist** d) {
    if (!nccl_unique_id || !d) return set_err(MM_E_ARG, "null argument");
    *d = nullptr;
    if (world < 1 || world > 8 || rank < 0 || rank >= world)
        return set_err(MM_E_ARG, "world must be in [1, 8] (one node) and rank in [0, world)");
    NcclApi* N = nccl();
    if (!N) return set_err(MM_E_NCCL, "libnccl.so.2 could not be loaded");
    mm_dist* D = new (std::nothrow) mm_dist;
    if (!D) return set_err(MM_E_ARG, "out of host memory");
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    cudaGetDevice(&D->dev);
    ncclResult_t r = N->commInitRank(&D->comm, world, id, rank);
    if (r != ncclSuccess) {
        delete D;
        return set_err(MM_E_NCCL, "ncclCommInitRank failed: %s", N->errorString(r));
    }
    D->rank = rank;
    D->world = world;
    *d = D;
    return MM_OK;
}

extern "C" void mm_dist_destroy(mm_dist* D) {
    if (!D) return;
    cudaDeviceSynchronize();
    for (int h = 0; h < 8; h++)
        if (D->peer_base[h]) cudaIpcCloseMemHandle(D->peer_base[h]);
    if (D->base) cudaFree(D->base);
    for (auto& kv : D->plans) mm_ntt_plan_destroy(kv.second);
    NcclApi* N = nccl();
    if (N && D->comm) N->commDestroy(D->comm);
    delete D;
}

extern "C" mm_status mm_dist_info(const mm_dist* D, int64_t out[4]) {
    if (!D || !out) return set_err(MM_E_ARG, "null argument");
    int v = 0;
    NcclApi* N = nccl();
    if (N && N->getVersion) N->getVersion(&v);
    out[0] = D->rank;
    out[1] = D->world;
    out[2] = D->p2p ? (int64_t)D->p2p_bytes : 0;
    out[3] = v;
    return MM_OK;
}

// Peer-memory transport: two receive buffers of `bytes` each plus a flag page
// in one cudaMalloc; handles exchanged with an NCCL all-gather; peers opened
// with cudaIpcOpenMemHandle.  Setup call: synchronises the device.
extern "C" mm_status mm_dist_p2p_enable(mm_dist* D, size_t bytes) {
    if (!D) return set_err(MM_E_ARG, "null argument");
    NcclApi* N = nccl();
    if (!N) return set_err(MM_E_NCCL, "libnccl.so.2 could not be loaded");
    std::lock_guard<std::mutex> g(D->mu);
    const int G = D->world;
    bytes = (bytes + 255) & ~(size_t)255;
    MM_CUDA_TRY(cudaDeviceSynchronize());
    for (int h = 0; h < 8; h++)
        if (D->peer_base[h]) {
            cudaIpcCloseMemHandle(D->peer_base[h]);
            D->peer_base[h] = nullptr;
        }
    if (D->base) {
        cudaFree(D->base);
        D->base = nullptr;
    }
    D->p2p = false;
    const size_t total = 2 * bytes + flag_page_bytes(G);
    MM_CUDA_TRY(cudaMalloc(&D->base, total));
    MM_CUDA_TRY(cudaMemset(D->base + 2 * bytes, 0, flag_page_bytes(G)));
    cudaIpcMemHandle_t mine;
    MM_CUDA_TRY(cudaIpcGetMemHandle(&mine, D->base));
    char* dbuf = nullptr;
    MM_CUDA_TRY(cudaMalloc(&dbuf, (size_t)(G + 1) * sizeof(mine)));
    MM_CUDA_TRY(cudaMemcpy(dbuf + G * sizeof(mine), &mine, sizeof(mine), cudaMemcpyHostToDevice));
    ncclResult_t r = N->allGather(dbuf + G * sizeof(mine), dbuf, sizeof(mine), ncclUint8, D->comm, 0);
    cudaIpcMemHandle_t all[8];
    cudaError_t e = r == ncclSuccess ? cudaMemcpy(all, dbuf, (size_t)G * sizeof(mine), cudaMemcpyDeviceToHost)
                                     : cudaSuccess;
    cudaFree(dbuf);
    if (r != ncclSuccess) return set_err(MM_E_NCCL, "handle all-gather failed: %s", N->errorString(r));
    if (e != cudaSuccess) return set_err(MM_E_CUDA, "handle copy failed: %s", cudaGetErrorString(e));
    for (int h = 0; h < G; h++) {
        char* b = D->base;
        if (h != D->rank) {
            void* q = nullptr;
            MM_CUDA_TRY(cudaIpcOpenMemHandle(&q, all[h], cudaIpcMemLazyEnablePeerAccess));
            b = (char*)q;
            D->peer_base[h] = b;
        }
        D->peer_recv[0][h] = b;
        D->peer_recv[1][h] = b + bytes;
        D->peer_flags.p[h] = (unsigned long long*)(b + 2 * bytes);
    }
    D->p2p_bytes = bytes;
    D->epoch = 0;
    D->p2p = true;
    MM_CUDA_TRY(cudaDeviceSynchronize());
    return MM_OK;
}

// Non-zero if a device-side wait of the peer transport timed out (a peer
// stopped responding): 1 + the flag slot.  Synchronises the device.
extern "C" mm_status mm_dist_p2p_status(mm_dist* D, uint64_t* slot) {
    if (!D || !slot) return set_err(MM_E_ARG, "null argument");
    *slot = 0;
    if (!D->p2p) return MM_OK;
    MM_CUDA_TRY(cudaDeviceSynchronize());
    MM_CUDA_TRY(cudaMemcpy(slot, D->base + 2 * D->p2p_bytes + 16 * D->world, 8, cudaMemcpyDeviceToHost));
    return MM_OK;
}

namespace mm {

struct DistGeom {
    uint64_t n1, n2, c1, r2;
    size_t es;
};
static mm_status dist_geom(const mm_dist* D, const mm_ntt_plan* plan, DistGeom* g, int* word_bits) {
    uint64_t info[6];
    mm_status s = mm_ntt_plan_info(plan, info);
    if (s != MM_OK) return s;
    if (info[5] != 1) return set_err(MM_E_ARG, "distributed transforms take batch-1 plans");
    if (info[2] != 2) return set_err(MM_E_UNSUPPORTED_SIZE, "the distributed transform needs a four-step plan");
    const int G = D->world;
    if (info[0] % G || info[1] % G) return set_err(MM_E_UNSUPPORTED_SIZE, "n1 = %llu, n2 = %llu not divisible by %d",
                                                   (unsigned long long)info[0], (unsigned long long)info[1], G);
    g->n1 = info[0];
    g->n2 = info[1];
    g->c1 = info[0] / G;
    g->r2 = info[1] / G;
    const int wb = (int)info[4];
    if (wb != 32 && wb != 64) return set_err(MM_E_ARG, "distributed transforms take 32- or 64-bit plans");
    g->es = wb == 32 ? 4 : 8;
    if (word_bits) *word_bits = wb;
    return MM_OK;
}

// equal-split all-to-all of `chunk` bytes per peer (grouped send / recv)
static mm_status all_to_all(mm_dist* D, const void* send, void* recv, size_t chunk, cudaStream_t st) {
    NcclApi* N = nccl();
    MM_NCCL_TRY(N->groupStart());
    for (int h = 0; h < D->world; h++) {
        MM_NCCL_TRY(N->send((const char*)send + h * chunk, chunk, ncclUint8, h, D->comm, st));
        MM_NCCL_TRY(N->recv((char*)recv + h * chunk, chunk, ncclUint8, h, D->comm, st));
    }
    MM_NCCL_TRY(N->groupEnd());
    return MM_OK;
}

static mm_status signal(mm_dist* D, int slot, unsigned long long v, cudaStream_t st) {
    {
        LaunchScope ls("dist_signal", st);
        k_dist_signal<<<1, 32, 0, st>>>(D->peer_flags, D->world, slot, v);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}
static mm_status wait_flags(mm_dist* D, int base, unsigned long long target, cudaStream_t st) {
    unsigned long long* own = D->peer_flags.p[D->rank];
    {
        LaunchScope ls("dist_wait", st);
        k_dist_wait<<<1, 32, 0, st>>>(own, base, D->world, target, own + 2 * D->world);
    }
    MM_LAUNCH_CHECK();
    return MM_OK;
}

}  // namespace mm

extern "C" mm_status mm_ntt_forward_dist(mm_dist* D, const mm_ntt_plan* plan, const void* local_in, void* local_out,
                                         void* stream) {
    if (!D || !plan || !local_in || !local_out) return set_err(MM_E_ARG, "null argument");
    DistGeom g;
    mm_status s = dist_geom(D, plan, &g, nullptr);
    if (s != MM_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int G = D->world, r = D->rank;
    const size_t blk = (size_t)g.n2 * g.c1 * g.es;       // bytes of one column (= row) block
    if (D->p2p && blk <= D->p2p_bytes) {
        std::lock_guard<std::mutex> lk(D->mu);
        const unsigned long long e = ++D->epoch;
        const int par = (int)(e & 1);
        if (e > 2 && (s = wait_flags(D, G, e - 2, st)) != MM_OK) return s;         // peers done with recv[par]
        if ((s = mm_ntt_fwd_cols_p2p(plan, local_in, D->peer_recv[par], G, r, (size_t)r * g.c1, g.c1, stream)) != MM_OK)
            return s;
        if ((s = signal(D, r, e, st)) != MM_OK) return s;                            // ready[r] = e at every peer
        if ((s = wait_flags(D, 0, e, st)) != MM_OK) return s;                        // all rows of my block arrived
        if ((s = mm_ntt_fwd_rows_seg(plan, D->peer_recv[par][r], local_out, (size_t)r * g.r2, g.r2, g.c1,
                                     g.r2 * g.c1, stream)) != MM_OK)
            return s;
        return signal(D, G + r, e, st);                                               // free[r] = e at every peer
    }
    void* ws = nullptr;
    MM_CUDA_TRY(alloc_async(&ws, 2 * blk, st));
    char* send = (char*)ws;
    char* recv = send + blk;
    if ((s = mm_ntt_fwd_cols(plan, local_in, send, (size_t)r * g.c1, g.c1, stream)) == MM_OK &&
        (s = all_to_all(D, send, recv, blk / G, st)) == MM_OK)
        s = mm_ntt_fwd_rows_seg(plan, recv, local_out, (size_t)r * g.r2, g.r2, g.c1, g.r2 * g.c1, stream);
    cudaFreeAsync(ws, st);
    return s;
}

extern "C" mm_status mm_ntt_inverse_dist(mm_dist* D, const mm_ntt_plan* plan, const void* local_in, void* local_out,
                                         void* stream) {
    if (!D || !plan || !local_in || !local_out) return set_err(MM_E_ARG, "null argument");
    DistGeom g;
    mm_status s = dist_geom(D, plan, &g, nullptr);
    if (s != MM_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int r = D->rank;
    const size_t blk = (size_t)g.n2 * g.c1 * g.es;
    void* ws = nullptr;
    MM_CUDA_TRY(alloc_async(&ws, 2 * blk, st));
    char* send = (char*)ws;
    char* recv = send + blk;
    if ((s = mm_ntt_inv_rows_seg(plan, local_in, send, (size_t)r * g.r2, g.r2, g.c1, g.r2 * g.c1, stream)) == MM_OK &&
        (s = all_to_all(D, send, recv, blk / D->world, st)) == MM_OK)
        s = mm_ntt_inv_cols(plan, recv, local_out, (size_t)r * g.c1, g.c1, stream);
    cudaFreeAsync(ws, st);
    return s;
}

extern "C" mm_status mm_int_mul_u16_dist(mm_dist* D, const uint16_t* a, size_t na, const uint16_t* b, size_t nb,
                                         uint16_t* local_c, void* stream) {
    if (!D || !a || !b || !local_c) return set_err(MM_E_ARG, "null argument");
    if (na == 0 || nb == 0) return set_err(MM_E_ARG, "empty operands");
    const uint64_t P = 0xFFFFFFFF00000001ull;
    const size_t mn = na < nb ? na : nb, nc = na + nb - 1, nout = na + nb;
    if ((unsigned __int128)mn * 0xFFFE0001ull >= P) return set_err(MM_E_SIZE_OVERFLOW, "min(na,nb)(2^16-1)^2 >= p");
    int k = 0;
    while ((1ull << k) < nc) k++;
    if (k < 14) k = 14;                                     // four-step plans start above one 2^13 pass
    if (k > 26) return set_err(MM_E_SIZE_OVERFLOW, "na + nb - 1 > 2^26");
    mm_ntt_plan* plan = nullptr;
    {
        std::lock_guard<std::mutex> lk(D->mu);
        auto it = D->plans.find(k);
        if (it != D->plans.end()) plan = it->second;
        else {
            const uint64_t w = hpowmod(7, (P - 1) >> k, P);   // 7 generates (Z/pZ)^*
            mm_status s = mm_ntt_plan_create(64, P, k, w, 1, &plan);
            if (s != MM_OK) return s;
            D->plans[k] = plan;
        }
    }
    DistGeom g;
    mm_status s = dist_geom(D, plan, &g, nullptr);
    if (s != MM_OK) return s;
    if (g.c1 < 4) return set_err(MM_E_UNSUPPORTED_SIZE, "column blocks need >= 4 columns (carry halo)");
    cudaStream_t st = (cudaStream_t)stream;
    const int G = D->world, r = D->rank;
    const size_t blk = (size_t)g.n2 * g.c1 * 8;
    // workspace: send, recvA, recvB, coefficients, halo out / in, aggregates
    const size_t halo = (size_t)g.n2 * 4 * 8, agg = (size_t)g.n2 * 4, agg_all = (size_t)G * g.n2 * 4;
    void* ws = nullptr;
    MM_CUDA_TRY(alloc_async(&ws, 4 * blk + 2 * halo + agg + agg_all + 256, st));
    char* send = (char*)ws;
    char* ra = send + blk;
    char* rb = ra + blk;
    uint64_t* coef = (uint64_t*)(rb + blk);
    uint64_t* hout = (uint64_t*)((char*)coef + blk);
    uint64_t* hin = hout + (size_t)g.n2 * 4;
    uint32_t* ag = (uint32_t*)(hin + (size_t)g.n2 * 4);
    uint32_t* ag_all = ag + g.n2;
    NcclApi* N = nccl();
    auto run = [&]() -> mm_status {
        mm_status q;
        const size_t col0 = (size_t)r * g.c1, row0 = (size_t)r * g.r2, segs = g.r2 * g.c1;
        if ((q = mm_ntt_fwd_cols_u16(plan, a, na, send, col0, g.c1, stream)) != MM_OK) return q;
        if ((q = all_to_all(D, send, ra, blk / G, st)) != MM_OK) return q;
        if ((q = mm_ntt_fwd_cols_u16(plan, b, nb, send, col0, g.c1, stream)) != MM_OK) return q;
        if ((q = all_to_all(D, send, rb, blk / G, st)) != MM_OK) return q;
        if ((q = mm_ntt_pmul_rows_seg(plan, ra, rb, send, row0, g.r2, g.c1, segs, stream)) != MM_OK) return q;
        if ((q = all_to_all(D, send, ra, blk / G, st)) != MM_OK) return q;
        if ((q = mm_ntt_inv_cols(plan, ra, coef, col0, g.c1, stream)) != MM_OK) return q;
        // carries (evaluation at 2^16): halo ring, chunk aggregates, all-gather, scan, apply
        if ((q = mm_carry_chunks_halo(coef, g.n2, g.c1, hout, stream)) != MM_OK) return q;
        if (G == 1) {
            MM_CUDA_TRY(cudaMemcpyAsync(hin, hout, halo, cudaMemcpyDeviceToDevice, st));
        } else {
            MM_NCCL_TRY(N->groupStart());
            MM_NCCL_TRY(N->send(hout, halo, ncclUint8, (r + 1) % G, D->comm, st));
            MM_NCCL_TRY(N->recv(hin, halo, ncclUint8, (r + G - 1) % G, D->comm, st));
            MM_NCCL_TRY(N->groupEnd());
        }
        if ((q = mm_carry_chunks_reduce(coef, hin, g.n2, g.c1, g.n1, col0, nc, nout, r == 0, ag, stream)) != MM_OK)
            return q;
        MM_NCCL_TRY(N->allGather(ag, ag_all, g.n2, ncclUint32, D->comm, st));
        if ((q = mm_carry_chunks_scan(ag_all, G, g.n2, stream)) != MM_OK) return q;
        return mm_carry_chunks_apply(coef, hin, g.n2, g.c1, g.n1, col0, nc, nout, r == 0, ag_all + (size_t)r * g.n2,
                                     local_c, stream);
    };
    s = run();
    cudaFreeAsync(ws, st);
    return s;
}

extern "C" mm_status mm_int_mul_u16_dist_layout(mm_dist* D, size_t na, size_t nb, uint64_t out[4]) {
    // {n1, n2, c1, k}: rank g's local_c is [n2][c1], limb j = r n1 + g c1 + i
    if (!D || !out || na == 0 || nb == 0) return set_err(MM_E_ARG, "bad argument");
    int k = 0;
    while ((1ull << k) < na + nb - 1) k++;
    if (k < 14) k = 14;
    if (k > 26) return set_err(MM_E_SIZE_OVERFLOW, "na + nb - 1 > 2^26");
    // the Goldilocks four-step split of ntt.cu (n1 = row length)
    uint64_t info[6];
    mm_ntt_plan* plan = nullptr;
    {
        std::lock_guard<std::mutex> lk(D->mu);
        auto it = D->plans.find(k);
        if (it != D->plans.end()) plan = it->second;
        else {
            const uint64_t P = 0xFFFFFFFF00000001ull;
            mm_status s = mm_ntt_plan_create(64, P, k, hpowmod(7, (P - 1) >> k, P), 1, &plan);
            if (s != MM_OK) return s;
            D->plans[k] = plan;
        }
    }
    mm_status s = mm_ntt_plan_info(plan, info);
    if (s != MM_OK) return s;
    out[0] = info[0];
    out[1] = info[1];
    out[2] = info[0] / D->world;
    out[3] = (uint64_t)k;
    return MM_OK;
}
