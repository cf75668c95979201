// Include shim for the reference header bfly/oracle.hpp (reference proj/include/bfly/oracle.hpp).
// classify_pairs / variance_bounds / OracleGuards / PairTypeCounts / VarianceBounds are the
// product's (the facade computes the pair types on the GPU). The enumeration helpers below
// are the reference tests' ground truth; they are TEST-SIDE code (oracle_support.cpp) and not
// part of libbfly_host.so.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "bfly_b200.hpp"

namespace bfly {

struct Butterfly {
  std::array<uint32_t, 2> left;
  std::array<uint32_t, 2> right;
};

inline bool operator==(const Butterfly& a, const Butterfly& b) {
  return a.left == b.left && a.right == b.right;
}

std::vector<Butterfly> enumerate_butterflies(const BipartiteGraph& g, const OracleGuards& guards = {});
uint64_t brute_force_count(const BipartiteGraph& g, const OracleGuards& guards = {});

}  // namespace bfly
