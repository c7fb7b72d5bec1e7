// gc_lru.h — bounded, thread-safe memo for the host-side constant caches (coefficients of
// eq. (19), O(1) operator fits).  Values are computed OUTSIDE the lock (a multiprecision
// eq. (19) can take milliseconds; other threads' gc_* calls must not wait on it) and
// inserted under it; lookups return copies, so eviction never invalidates a caller's data.
#pragma once

#include <cstddef>
#include <map>
#include <mutex>
#include <utility>

namespace gc {

template <typename K, typename V, size_t Cap = 64>
class LruMemo {
 public:
  template <typename F>
  V get(const K& key, F&& compute) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto it = map_.find(key);
      if (it != map_.end()) {
        it->second.second = ++clock_;
        return it->second.first;
      }
    }
    V v = compute();                       // no lock held
    std::lock_guard<std::mutex> lk(mu_);
    auto it = map_.find(key);
    if (it != map_.end()) return it->second.first;   // another thread inserted it meanwhile
    if (map_.size() >= Cap) {              // evict the least recently used entry
      auto old = map_.begin();
      for (auto j = map_.begin(); j != map_.end(); ++j)
        if (j->second.second < old->second.second) old = j;
      map_.erase(old);
    }
    map_.emplace(key, std::make_pair(v, ++clock_));
    return v;
  }

 private:
  std::mutex mu_;
  std::map<K, std::pair<V, unsigned long long>> map_;
  unsigned long long clock_ = 0;
};

}  // namespace gc
