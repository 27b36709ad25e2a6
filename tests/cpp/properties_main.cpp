// SPEC acceptance properties written against the reference
// headers only, so the same program builds against the reference and against
// ours (tests/test_cpp_properties.py requires byte-identical output):
//  1. Alg. 1 over 1,000 random censuses: ratios sum to exactly 1 and each is
//     s*c/total exactly; Alg. 2 never plans more than the available bytes nor
//     more buffers than the census holds (gpu + cpu <= count).
//  9. BufferPool model-based test: 100,000 random acquire / release /
//     find_victim / set_designated / occupants operations against a simple
//     model: chunks disjoint and covering the region, FIFO free lists, double
//     release detected, occupied bytes consistent.
// Prints a digest of every observable result; exits non-zero on a violated
// property.
#include <cstdint>
#include <cstdio>
#include <deque>
#include <iostream>
#include <map>
#include <random>
#include <set>
#include <vector>

#include "tencache/bufpool.hpp"

using namespace tencache;

static std::uint64_t digest = 1469598103934665603ull;
static void mix(std::uint64_t v) {
  digest ^= v;
  digest *= 1099511628211ull;
}
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("property violated: %s (line %d)\n", #c, __LINE__); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main() {
  std::mt19937_64 rng(2024);
  const std::uint64_t sizes[] = {512, 1024, 4096, 65536, 1u << 20, 3u << 20, 33574912};
  // ---- 1. Alg. 1 / Alg. 2 over 1,000 random censuses
  for (int k = 0; k < 1000; ++k) {
    TensorCensus tc;
    const int classes = 1 + static_cast<int>(rng() % 6);
    for (int c = 0; c < classes; ++c) tc[sizes[rng() % 7] + (rng() % 3) * 4096] += 1 + rng() % 50;
    const SizeDistribution sd = size_distribution(tc);
    Rat sum = rat_of(0);
    std::uint64_t total = 0;
    for (const auto& [s, c] : tc) total += s * c;
    CHECK(sd.total_size == total);
    for (const auto& [s, c] : tc) {
      CHECK(sd.ratios.at(s) == Rat(BigInt(s * c), BigInt(total)));
      sum += sd.ratios.at(s);
    }
    CHECK(sum == rat_of(1));
    const std::uint64_t gpu = rng() % (total + 1), cpu = rng() % (total + 1);
    const BufferPlan p = plan_buffers(tc, sd, gpu, cpu);
    CHECK(p.gpu_planned_bytes() <= gpu);
    CHECK(p.cpu_planned_bytes() <= cpu);
    for (const auto& [s, c] : tc) {
      const std::uint64_t g = p.gpu_counts.count(s) ? p.gpu_counts.at(s) : 0;
      const std::uint64_t h = p.cpu_counts.count(s) ? p.cpu_counts.at(s) : 0;
      CHECK(g + h <= c);
      mix(s);
      mix(g);
      mix(h);
    }
  }
  std::printf("alg1/alg2 1000 censuses ok digest %016llx\n", static_cast<unsigned long long>(digest));

  // ---- 9. BufferPool against a model, 100,000 operations
  std::map<std::uint64_t, std::uint64_t> counts{{512, 7}, {4096, 5}, {65536, 3}, {1u << 20, 2}};
  BufferPool pool = BufferPool::build(Tier::Cpu, counts);
  std::uint64_t region = 0;
  for (const auto& [s, n] : counts) region += s * n;
  CHECK(pool.region_bytes() == region);
  {  // layout: ascending class, then index; contiguous from 0, disjoint
    std::uint64_t off = 0;
    for (const Chunk& c : pool.chunks()) {
      CHECK(c.offset == off);
      off += c.size;
    }
    CHECK(off == region);
  }
  std::map<std::uint64_t, std::deque<std::uint32_t>> free_model;
  for (const Chunk& c : pool.chunks()) free_model[c.size].push_back(c.buffer_id);
  std::map<std::uint32_t, TensorId> occ_model;
  std::set<std::uint32_t> designated_model;
  std::uint64_t occ_bytes = 0;
  TensorId next_tensor = 1;
  std::vector<std::uint64_t> class_list;
  for (const auto& [s, n] : counts) class_list.push_back(s);
  int double_release_caught = 0, unknown_class_caught = 0;
  for (int op = 0; op < 100000; ++op) {
    const int kind = static_cast<int>(rng() % 6);
    const std::uint64_t s = class_list[rng() % class_list.size()];
    if (kind <= 1) {  // acquire
      const auto b = pool.acquire(s, next_tensor);
      if (free_model[s].empty()) {
        CHECK(!b.has_value());
      } else {
        CHECK(b.has_value() && *b == free_model[s].front());  // FIFO pop
        free_model[s].pop_front();
        occ_model[*b] = next_tensor;
        occ_bytes += s;
        CHECK(pool.buffer_of(next_tensor) == b);
      }
      mix(b ? *b : 0xffffffffu);
      ++next_tensor;
    } else if (kind == 2) {  // release (sometimes a double release)
      const std::uint32_t b = static_cast<std::uint32_t>(rng() % pool.chunks().size());
      const bool occupied = occ_model.count(b) != 0;
      try {
        pool.release(b);
        CHECK(occupied);
        free_model[pool.chunk(b).size].push_back(b);  // FIFO push back
        occ_bytes -= pool.chunk(b).size;
        occ_model.erase(b);
        designated_model.erase(b);
      } catch (const PoolError&) {
        CHECK(!occupied);
        ++double_release_caught;
      }
      mix(b);
    } else if (kind == 3) {  // find_victim (lowest offset, designated preferred when asked)
      const bool pref = rng() % 2;
      const auto v = pool.find_victim(s, pref);
      std::optional<std::pair<std::uint32_t, TensorId>> want;
      for (const auto& [b, t] : occ_model)  // buffer ids ascend with offsets within a class
        if (pool.chunk(b).size == s && (!pref || designated_model.count(b))) {
          want = std::make_pair(b, t);
          break;
        }
      if (pref && !want)
        for (const auto& [b, t] : occ_model)
          if (pool.chunk(b).size == s) {
            want = std::make_pair(b, t);
            break;
          }
      mix(v ? v->first : 0xfffffffeu);
      mix(want ? want->first : 0xfffffffeu);
    } else if (kind == 4) {  // designate an occupied buffer
      if (!occ_model.empty()) {
        auto it = occ_model.begin();
        std::advance(it, static_cast<long>(rng() % occ_model.size()));
        pool.set_designated(it->first, true);
        designated_model.insert(it->first);
        mix(it->first);
      }
    } else {  // occupants + an unknown class
      const auto occ = pool.occupants(s, false);
      std::size_t n = 0;
      for (const auto& [b, t] : occ_model)
        if (pool.chunk(b).size == s) ++n;
      CHECK(occ.size() == n);
      for (const auto& [b, t] : occ) {
        CHECK(occ_model.at(b) == t);
        mix(b);
      }
      try {
        (void)pool.acquire(777, next_tensor);
      } catch (const PoolError&) {
        ++unknown_class_caught;
      }
    }
    CHECK(pool.occupied_bytes() == occ_bytes);
    for (const auto& [cs, fl] : free_model) CHECK(pool.free_count(cs) == fl.size());
  }
  std::printf("pool 100000 ops ok: double releases caught %d, unknown class %d, digest %016llx\n",
              double_release_caught, unknown_class_caught, static_cast<unsigned long long>(digest));
  return 0;
}
