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
