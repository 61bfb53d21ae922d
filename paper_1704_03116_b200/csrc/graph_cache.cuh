// graph_cache.cuh -- bounded cache of instantiated CUDA graphs (host side).
//
// The run loops (dope_admm_run, dope_f_admm_run, dope_g_admm_run,
// dope_sharded_run) capture `iters` iterations once and replay the graph.  A
// graph bakes in the device pointers of the lattice description, so the key
// is the description's exact bytes plus the iteration count; an entry may also
// name an owner (a communicator) whose destruction must drop it.  Each cache
// holds at most `cap` graphs (DOPE_GRAPH_CACHE, default 8) and destroys the
// least recently used one beyond that -- cudaGraphExecDestroy on an in-flight
// graph frees it once it completes.  All caches register themselves so that
// dope_graph_cache_entries / dope_graph_cache_clear see every one.
#pragma once
#include <cuda_runtime.h>
#include <stdlib.h>

#include <list>
#include <mutex>
#include <string>
#include <vector>

namespace dope {

class GraphCache;

// one registry for the whole library: an inline function's static is shared
// by every translation unit of the .so
inline std::vector<GraphCache *> &graph_cache_registry() {
    static std::vector<GraphCache *> r;
    return r;
}
inline std::mutex &graph_cache_registry_mutex() {
    static std::mutex m;
    return m;
}

class GraphCache {
  public:
    GraphCache() {
        const char *e = getenv("DOPE_GRAPH_CACHE");
        cap_ = e ? (size_t)atoi(e) : 8;
        if (cap_ < 1) cap_ = 1;
        std::lock_guard<std::mutex> lk(graph_cache_registry_mutex());
        graph_cache_registry().push_back(this);
    }
    GraphCache(const GraphCache &) = delete;
    GraphCache &operator=(const GraphCache &) = delete;

    cudaGraphExec_t find(const std::string &key) {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = lru_.begin(); it != lru_.end(); ++it)
            if (it->key == key) {
                lru_.splice(lru_.begin(), lru_, it);   // most recently used first
                return it->exec;
            }
        return nullptr;
    }

    void put(const std::string &key, cudaGraphExec_t exec, const void *owner = nullptr) {
        std::lock_guard<std::mutex> lk(mu_);
        lru_.push_front(Entry{key, exec, owner});
        while (lru_.size() > cap_) {
            cudaGraphExecDestroy(lru_.back().exec);
            lru_.pop_back();
        }
    }

    // drop every graph captured against `owner` (e.g. a destroyed communicator)
    void erase_owner(const void *owner) {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = lru_.begin(); it != lru_.end();) {
            if (it->owner == owner) {
                cudaGraphExecDestroy(it->exec);
                it = lru_.erase(it);
            } else {
                ++it;
            }
        }
    }

    size_t size() {
        std::lock_guard<std::mutex> lk(mu_);
        return lru_.size();
    }

    void clear() {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto &e : lru_) cudaGraphExecDestroy(e.exec);
        lru_.clear();
    }

  private:
    struct Entry {
        std::string key;
        cudaGraphExec_t exec;
        const void *owner;
    };
    std::mutex mu_;
    std::list<Entry> lru_;
    size_t cap_ = 8;
};

inline int64_t graph_cache_entries_all() {
    std::lock_guard<std::mutex> lk(graph_cache_registry_mutex());
    int64_t n = 0;
    for (GraphCache *c : graph_cache_registry()) n += (int64_t)c->size();
    return n;
}

inline void graph_cache_clear_all() {
    std::lock_guard<std::mutex> lk(graph_cache_registry_mutex());
    for (GraphCache *c : graph_cache_registry()) c->clear();
}

}  // namespace dope
