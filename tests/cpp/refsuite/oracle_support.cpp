// oracle_support.cpp -- TEST-SIDE ground truth for the reference's unit tests compiled against
// the facade: butterflies listed by definition (every left pair a < b, every pair of common
// right neighbours i < j), as the reference's enumeration oracle specifies
// (oracle.hpp:20-33, oracle.cpp:37-58). It reads the graph only through the public accessors
// (neighbors() on the facade's host mirror), never through the counting path under test.
#include <algorithm>
#include <iterator>
#include <string>

#include "bfly/oracle.hpp"

namespace bfly {
namespace {

void guard_sides(const BipartiteGraph& g, const OracleGuards& guards) {
  if (g.left_count() > guards.max_side || g.right_count() > guards.max_side)
    throw SizeGuardError("oracle guard: side exceeds " + std::to_string(guards.max_side) +
                         " vertices (raise the guard to override)");
}

std::vector<uint32_t> common_right(const BipartiteGraph& g, uint32_t a, uint32_t b) {
  auto na = g.neighbors(Side::Left, a), nb = g.neighbors(Side::Left, b);
  std::vector<uint32_t> out;
  std::set_intersection(na.begin(), na.end(), nb.begin(), nb.end(), std::back_inserter(out));
  return out;
}

}  // namespace

std::vector<Butterfly> enumerate_butterflies(const BipartiteGraph& g, const OracleGuards& guards) {
  guard_sides(g, guards);
  std::vector<Butterfly> out;
  for (uint32_t a = 0; a < g.left_count(); ++a)
    for (uint32_t b = a + 1; b < g.left_count(); ++b) {
      const auto c = common_right(g, a, b);
      for (size_t i = 0; i < c.size(); ++i)
        for (size_t j = i + 1; j < c.size(); ++j) out.push_back({{a, b}, {c[i], c[j]}});
    }
  return out;
}

uint64_t brute_force_count(const BipartiteGraph& g, const OracleGuards& guards) {
  guard_sides(g, guards);
  uint64_t total = 0;
  for (uint32_t a = 0; a < g.left_count(); ++a)
    for (uint32_t b = a + 1; b < g.left_count(); ++b)
      total = checked_add(total, choose2(common_right(g, a, b).size()));
  return total;
}

}  // namespace bfly
