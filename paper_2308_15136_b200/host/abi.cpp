#include "abi.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fodg/b200.hpp"

namespace fodg::b200 {

void check(int rc) {
    if (rc == CAGRA_OK) return;
    const std::string msg = cagra_last_error();
    switch (rc) {
        case CAGRA_ERR_USAGE: throw UsageError(msg);
        case CAGRA_ERR_FORMAT: throw FormatError(msg);
        case CAGRA_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error("cagra: " + msg);
    }
}

int device() {
    const char* e = std::getenv("CAGRA_DEVICE");
    return e ? std::atoi(e) : 0;
}

std::vector<int> devices() {
    // CAGRA_DEVICES=0,1,2,3 spreads batch_search / exact_knn_graph over those
    // GPUs (query-sharded replicas, row-sharded kNN build); default: device()
    std::vector<int> out;
    if (const char* e = std::getenv("CAGRA_DEVICES")) {
        const char* s = e;
        while (*s) {
            char* end = nullptr;
            const long v = std::strtol(s, &end, 10);
            if (end == s) break;
            out.push_back(static_cast<int>(v));
            s = *end == ',' ? end + 1 : end;
        }
    }
    if (out.empty()) out.push_back(device());
    return out;
}

bool fast_distances() {
    const char* e = std::getenv("CAGRA_FAST_DISTANCES");
    return !(e && e[0] == '0');
}

unsigned device_sm_count() {
    static int cached = -1;
    if (cached < 0) {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device()) != cudaSuccess ||
            sms <= 0)
            sms = 148;  // B200
        cached = sms;
    }
    return static_cast<unsigned>(cached);
}

namespace {

// ---- content hash ----------------------------------------------------------
// The reference reads its `const Graph&, const Dataset&` afresh on every call,
// so the device copy may be reused only while the host contents are exactly
// the ones uploaded.  Every cached lookup therefore hashes the WHOLE of both
// buffers (no sampling): four independent 64-bit multiply-rotate lanes per
// chunk, chunks spread over host threads for large buffers (memory-bound,
// tens of GB/s), folded in chunk order so the value is thread-count independent.
inline std::uint64_t rotl(std::uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

std::uint64_t hash_chunk(const unsigned char* p, std::size_t bytes, std::uint64_t seed) {
    constexpr std::uint64_t P1 = 0x9e3779b185ebca87ull, P2 = 0xc2b2ae3d27d4eb4full;
    std::uint64_t a = seed ^ P1, b = seed ^ P2, c = seed + P1, d = seed - P2;
    std::size_t i = 0;
    for (; i + 32 <= bytes; i += 32) {
        std::uint64_t w[4];
        std::memcpy(w, p + i, 32);
        a = rotl(a ^ (w[0] * P2), 31) * P1;
        b = rotl(b ^ (w[1] * P2), 31) * P1;
        c = rotl(c ^ (w[2] * P2), 31) * P1;
        d = rotl(d ^ (w[3] * P2), 31) * P1;
    }
    std::uint64_t h = rotl(a, 1) + rotl(b, 7) + rotl(c, 12) + rotl(d, 18);
    for (; i < bytes; ++i) h = (h ^ p[i]) * P1;
    return (h ^ (h >> 29)) * P2 ^ bytes;
}

std::uint64_t content_hash(const void* p, std::size_t bytes) {
    const auto* b = static_cast<const unsigned char*>(p);
    constexpr std::size_t kChunk = 8u << 20;
    const std::size_t chunks = (bytes + kChunk - 1) / kChunk;
    if (chunks <= 1) return hash_chunk(b, bytes, 0x5eed);
    std::vector<std::uint64_t> part(chunks);
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const unsigned nt = static_cast<unsigned>(std::min<std::size_t>(hw, chunks));
    auto work = [&](unsigned t) {
        for (std::size_t c = t; c < chunks; c += nt) {
            const std::size_t lo = c * kChunk, len = std::min(kChunk, bytes - lo);
            part[c] = hash_chunk(b + lo, len, c);
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    return hash_chunk(reinterpret_cast<const unsigned char*>(part.data()), 8 * chunks, bytes);
}

bool trust_identity() {
    // CAGRA_INDEX_CACHE=identity: the caller promises not to mutate a searched
    // Graph/Dataset in place (or calls invalidate_index_cache() after doing so);
    // lookups then match on addresses and shapes only and skip the hash
    const char* e = std::getenv("CAGRA_INDEX_CACHE");
    return e && std::strcmp(e, "identity") == 0;
}

struct CacheEntry {
    const void* data;
    const void* ids;
    std::uint32_t n, dim, degree;
    std::uint64_t h_data, h_ids;
    cagra_index* ix;     // single device, or
    cagra_mindex* mx;    // the CAGRA_DEVICES set
    std::vector<int> devs;
};

void destroy(CacheEntry& e) {
    if (e.ix) cagra_index_destroy(e.ix);
    if (e.mx) cagra_mindex_destroy(e.mx);
}

std::mutex g_mu;
std::list<CacheEntry> g_cache;  // most recent first
constexpr std::size_t kMaxCached = 4;

}  // namespace

namespace {

// Looks up (or uploads) the device copy of (graph, ds) for `devs`: one
// device -> cagra_index, several -> a replicated cagra_mindex.
CacheEntry& entry_for(const Graph& graph, const Dataset& ds, const std::vector<int>& devs) {
    const bool identity = trust_identity();
    const std::uint64_t hd = identity ? 0 : content_hash(ds.raw(), 4ull * ds.size() * ds.dim());
    const std::uint64_t hi = identity ? 0 : content_hash(graph.ids.data(), 4ull * graph.ids.size());
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (it->data == ds.raw() && it->ids == graph.ids.data() && it->n == ds.size() &&
            it->dim == ds.dim() && it->degree == graph.degree && it->devs == devs &&
            (identity || (it->h_data == hd && it->h_ids == hi))) {
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front();
        }
    }
    CacheEntry e{ds.raw(), graph.ids.data(), ds.size(), ds.dim(), graph.degree, hd, hi,
                 nullptr, nullptr, devs};
    if (devs.size() == 1)
        check(cagra_index_create(ds.raw(), ds.size(), ds.dim(), graph.ids.data(), graph.degree,
                                 devs[0], &e.ix));
    else
        check(cagra_mindex_create(ds.raw(), ds.size(), ds.dim(), graph.ids.data(), graph.degree,
                                  devs.data(), static_cast<std::uint32_t>(devs.size()),
                                  CAGRA_SHARD_REPLICATE, &e.mx));
    g_cache.push_front(e);
    while (g_cache.size() > kMaxCached) {
        destroy(g_cache.back());
        g_cache.pop_back();
    }
    return g_cache.front();
}

}  // namespace

cagra_index* index_for(const Graph& graph, const Dataset& ds) {
    std::lock_guard<std::mutex> lock(g_mu);
    return entry_for(graph, ds, {device()}).ix;
}

void with_index(const Graph& graph, const Dataset& ds,
                const std::function<void(cagra_index*, cagra_mindex*)>& search) {
    const std::vector<int> devs = devices();
    if (trust_identity()) {
        cagra_index* ix = nullptr;
        cagra_mindex* mx = nullptr;
        {
            std::lock_guard<std::mutex> lock(g_mu);
            CacheEntry& e = entry_for(graph, ds, devs);
            ix = e.ix;
            mx = e.mx;
        }
        search(ix, mx);
        return;
    }
    // a copy matching by address and shape is searched while its contents are
    // re-hashed on host threads (the previous hashes are in the entry)
    cagra_index* ix = nullptr;
    cagra_mindex* mx = nullptr;
    std::uint64_t want_d = 0, want_i = 0;
    {
        std::lock_guard<std::mutex> lock(g_mu);
        for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
            if (it->data == ds.raw() && it->ids == graph.ids.data() && it->n == ds.size() &&
                it->dim == ds.dim() && it->degree == graph.degree && it->devs == devs) {
                g_cache.splice(g_cache.begin(), g_cache, it);
                ix = it->ix;
                mx = it->mx;
                want_d = it->h_data;
                want_i = it->h_ids;
                break;
            }
        }
    }
    if (ix || mx) {
        std::uint64_t hd = 0, hi = 0;
        std::thread hasher([&] {
            hd = content_hash(ds.raw(), 4ull * ds.size() * ds.dim());
            hi = content_hash(graph.ids.data(), 4ull * graph.ids.size());
        });
        try {
            search(ix, mx);
        } catch (...) {
            hasher.join();
            throw;
        }
        hasher.join();
        if (hd == want_d && hi == want_i) return;
        // contents changed in place: drop the stale copy, upload, search again
        std::lock_guard<std::mutex> lock(g_mu);
        for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
            if (it->ix == ix && it->mx == mx) {
                destroy(*it);
                g_cache.erase(it);
                break;
            }
    }
    {
        std::lock_guard<std::mutex> lock(g_mu);
        CacheEntry& e = entry_for(graph, ds, devs);
        ix = e.ix;
        mx = e.mx;
    }
    search(ix, mx);
}

cagra_mindex* mindex_for(const Graph& graph, const Dataset& ds) {
    std::lock_guard<std::mutex> lock(g_mu);
    return entry_for(graph, ds, devices()).mx;
}

void invalidate_index_cache() {
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto& e : g_cache) destroy(e);
    g_cache.clear();
}

std::uint64_t host_content_hash(const void* p, std::size_t bytes) { return content_hash(p, bytes); }

}  // namespace fodg::b200
