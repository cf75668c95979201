/* synth.h -- seeded synthetic bipartite edge lists for the BASELINE.json configs.
 * Stand-ins for the paper's KONECT graphs (not in this container). Host C++, threads.
 * Candidate t uses counter-based draws derive_seed(seed_side, t) (rng.hpp:18-31 mixers),
 * so output is independent of the thread count. Edges are emitted in draw order, keeping
 * the first occurrence of every (l, r) pair, until m distinct pairs exist. */
#ifndef BFLY_SYNTH_H
#define BFLY_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* uniform pairs over [0,U) x [0,V) (config 1) */
int bfly_synth_uniform(uint32_t U, uint32_t V, uint64_t m, uint64_t seed, uint32_t* l,
                       uint32_t* r);
/* Chung-Lu: endpoint i drawn with probability proportional to (i+1)^(-1/(gamma-1)) by
 * inverse CDF on double prefix sums. max_degree > 0 rejects draws whose endpoint already
 * has max_degree distinct neighbours (config 3's realised-degree cap). */
int bfly_synth_chung_lu(uint32_t U, uint32_t V, uint64_t m, double gamma_u, double gamma_v,
                        uint32_t max_degree, uint64_t seed, uint32_t* l, uint32_t* r);
#ifdef __cplusplus
}
#endif
#endif
