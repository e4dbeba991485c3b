// common.cu -- status handling and the 32-bit modulus context.
#include "common.h"
#include <stdlib.h>
#include <string.h>
#include <new>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>
#include <map>

namespace mm {

static thread_local char g_err[512] = "";

mm_status set_err(mm_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

int num_sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

static std::mutex g_pool_mu;
static std::map<int, cudaMemPool_t> g_pools;
static cudaMemPool_t lib_pool(int dev) {
    std::lock_guard<std::mutex> g(g_pool_mu);
    auto it = g_pools.find(dev);
    if (it != g_pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    g_pools[dev] = pool;
    return pool;
}
cudaError_t alloc_async(void **p, size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = lib_pool(dev);
    if (!pool) return cudaMallocAsync(p, bytes, st);
    return cudaMallocFromPoolAsync(p, bytes, pool, st);
}
void trim_pool() {
    std::lock_guard<std::mutex> g(g_pool_mu);
    for (auto &kv : g_pools) cudaMemPoolTrimTo(kv.second, 0);
}

bool debug_checks() {
    const char *e = getenv("MMNTT_DEBUG");
    return e && e[0] == '1';
}

bool hprime(uint64_t n) {
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (uint64_t q : small) {
        if (n == q) return true;
        if (n % q == 0) return false;
    }
    uint64_t d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (uint64_t a : small) {
        uint64_t x = hpowmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s; r++) {
            x = hmulmod(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

// ---- MMNTT_DEBUG input range checks (header conventions): residues of rows
// [rows][len] at row stride ld must be canonical -- u32 / u64 below p, FP64
// (word_bits 52) integral in [0, p).  One counting kernel, then a stream sync.
template <class T>
__global__ void k_rows_range(const T* __restrict__ x, long long rows, long long len, long long ld, uint64_t p,
                             unsigned long long* bad) {
    unsigned long long local = 0;
    const long long n = rows * len;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / len, j = i - r * len;
        const T v = x[r * ld + j];
        if constexpr (sizeof(T) == 8 && T(0.5) != T(0)) {
            local += !(v >= 0.0 && v < (double)p && floor(v) == v);
        } else {
            local += (uint64_t)v >= p;
        }
    }
    if (local) atomicAdd(bad, local);
}

mm_status check_rows(const void *x, int word_bits, size_t rows, size_t len, size_t ld, uint64_t p, cudaStream_t st) {
    if (!x || !rows || !len) return MM_OK;
    unsigned long long *d = nullptr, h = 0;
    MM_CUDA_TRY(alloc_async((void **)&d, sizeof(*d), st));
    MM_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(*d), st));
    {
        LaunchScope ls("debug_range_check", st);
        const int grid = num_sms() * 4;
        if (word_bits == 32)
            k_rows_range<uint32_t><<<grid, 256, 0, st>>>((const uint32_t *)x, (long long)rows, (long long)len,
                                                         (long long)ld, p, d);
        else if (word_bits == 64)
            k_rows_range<uint64_t><<<grid, 256, 0, st>>>((const uint64_t *)x, (long long)rows, (long long)len,
                                                         (long long)ld, p, d);
        else
            k_rows_range<double><<<grid, 256, 0, st>>>((const double *)x, (long long)rows, (long long)len,
                                                       (long long)ld, p, d);
    }
    MM_LAUNCH_CHECK();
    MM_CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    MM_CUDA_TRY(cudaFreeAsync(d, st));
    MM_CUDA_TRY(cudaStreamSynchronize(st));
    if (h) return set_err(MM_E_RANGE, "%llu input residues outside [0, p)", h);
    return MM_OK;
}

static std::atomic<unsigned long long> g_launches{0};
static std::atomic<int> g_prof{0};
static std::mutex g_prof_mu;
struct ProfRec { std::string name; cudaEvent_t a, b; };
static std::vector<ProfRec> g_recs;

LaunchScope::LaunchScope(const char *n, cudaStream_t s) : name(n), st(s), slot(-1) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (g_prof.load(std::memory_order_relaxed)) {
        ProfRec r{n, nullptr, nullptr};
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        cudaEventRecord(r.a, s);
        std::lock_guard<std::mutex> g(g_prof_mu);
        slot = (int)g_recs.size();
        g_recs.push_back(r);
    }
}
LaunchScope::~LaunchScope() {
    if (slot >= 0) {
        std::lock_guard<std::mutex> g(g_prof_mu);
        cudaEventRecord(g_recs[slot].b, st);
    }
}

}  // namespace mm

extern "C" unsigned long long mm_launch_count(void) { return mm::g_launches.load(); }

static std::map<std::string, std::pair<unsigned long long, double>> g_agg;

extern "C" void mm_prof_enable(int on) {
    using namespace mm;
    if (on) {
        std::lock_guard<std::mutex> g(g_prof_mu);
        g_agg.clear();
    }
    g_prof.store(on ? 1 : 0);
}

extern "C" int mm_prof_collect(char *buf, size_t len) {
    using namespace mm;
    std::lock_guard<std::mutex> g(g_prof_mu);
    auto &agg = g_agg;
    for (auto &r : g_recs) {
        float ms = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto &e = agg[r.name];
        e.first += 1;
        e.second += ms;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_recs.clear();
    std::string out;
    for (auto &kv : agg) {
        char line[256];
        snprintf(line, sizeof line, "%s %llu %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
        out += line;
    }
    if (buf && len) {
        snprintf(buf, len, "%s", out.c_str());
    }
    return (int)out.size();
}

extern "C" const char *mm_last_error(void) { return mm::g_err; }
extern "C" const char *mm_version(void) { return "mmntt 0.1 (sm_100a)"; }
