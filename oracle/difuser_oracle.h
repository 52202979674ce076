/*
 * difuser_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's sketch-IM hot path (DiFuseR CPU
 * reference, /root/reference/proj), used exclusively as the parity CHECKER by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  It is never
 * linked into, loaded by or called from the product library
 * (paper_2410_14047_b200/).  Every function cites the reference file:line it
 * restates.  Parity pinning: the restatement is checked against the reference's
 * own golden vectors (tests/data/hash_vectors.csv, test_hash.cpp KATs) and
 * against fixtures produced by the compiled reference (tests/golden/, made by
 * oracle/make_golden.py through oracle/_ref).
 */
#ifndef DIFUSER_ORACLE_H
#define DIFUSER_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- L0 primitives (proj/include/difuser/hash.hpp) ---------------------- */
uint64_t dor_fmix64(uint64_t k);
uint64_t dor_splitmix64_at(uint64_t seed, uint64_t i);
void dor_murmur3_pair(uint64_t a, uint64_t b, uint64_t out[2]);
uint32_t dor_edge_hash(uint64_t u, uint64_t v);
uint64_t dor_register_hash(uint64_t jkey, uint64_t v);
uint32_t dor_random_value_at(uint64_t seed, uint32_t r);
uint32_t dor_to_fixed_point(double w);

/* ---- weights (proj/src/graph.cpp:247-258) ------------------------------- */
void dor_weights_const(double p, uint64_t m, uint32_t *w);
void dor_weights_wc(uint32_t n, uint64_t m, const uint64_t *offsets,
                    const uint32_t *adj, uint32_t *w);

/* ---- FASST plan (proj/src/fasst.cpp:21-48) ------------------------------ */
int dor_make_plan(uint32_t r, uint32_t mu, int fasst, uint64_t seed,
                  uint32_t *x_sorted, uint32_t *order, int *degraded);

/* ---- device graph with baked masks (proj/src/fasst.cpp:50-88) ----------
 * Returns m_tau; out arrays sized n+1, m, m*words (caller-owned). */
uint64_t dor_device_graph(uint32_t n, const uint64_t *offsets,
                          const uint32_t *adj, const uint32_t *ehash,
                          const uint32_t *w, const uint32_t *xs,
                          uint32_t j_local, uint64_t *d_offsets,
                          uint32_t *d_adj, uint64_t *d_mask);

/* ---- sketch state (proj/src/sketch.cpp) --------------------------------- */
void dor_fill(uint32_t n, uint32_t j_local, uint32_t j_offset, uint64_t key,
              int8_t *regs);
double dor_row_score(const int8_t *row, uint32_t j_local);

/* ---- engine (proj/src/engine.cpp) ---------------------------------------
 * Jacobi simulate to convergence; returns sweep count, or -1 when `cap`
 * sweeps did not converge (the reference throws runtime_error). */
int dor_simulate(uint32_t n, const uint64_t *d_offsets, const uint32_t *d_adj,
                 const uint64_t *d_mask, uint32_t j_local, int8_t *regs,
                 int cap);
/* commit_seed + cascade; vis is n*words u64 (bitset mirror of VISITED);
 * returns the number of registers newly marked VISITED. */
uint64_t dor_commit_cascade(uint32_t n, const uint64_t *d_offsets,
                            const uint32_t *d_adj, const uint64_t *d_mask,
                            uint32_t j_local, int8_t *regs, uint64_t *vis,
                            uint32_t seed);

/* ---- FASST analytics (proj/src/fasst.cpp:90-168): duplication histogram
 * dup_count[mu+1], per-chunk edge loads[mu], fill-rate live lanes / batches
 * over xfill (X sorted for FASST, generation order for naive). */
void dor_fasst_stats(uint64_t m, const uint32_t *ehash, const uint32_t *w,
                     const uint32_t *xs, const uint32_t *xfill, uint32_t r,
                     uint32_t mu, uint64_t *dup_count, uint64_t *loads,
                     uint64_t *live_lanes, uint64_t *batches);

/* ---- full greedy run (proj/src/runtime.cpp:37-179), mu simulated devices
 * executed one after another.  `w` is the fixed-point weight array already
 * assigned (apply_weights).  Outputs: seeds_dense[k], traj[k],
 * rebuild_rounds[k] (first *n_rebuilds valid), flags, counters[3] =
 * {reduced_elements, broadcast_elements, barriers}.  Returns 0, or a negative
 * code: -1 invalid argument, -2 simulate cap exceeded, -3 out of memory. */
int dor_run(uint32_t n, uint64_t m, const uint64_t *offsets,
            const uint32_t *adj, const uint32_t *w, uint32_t k, uint32_t r,
            uint32_t mu, int fasst, double rebuild_eps, uint64_t seed,
            int sim_cap, uint32_t *seeds_dense, double *traj,
            uint32_t *rebuild_rounds, uint32_t *n_rebuilds, int *saturated,
            int *degraded, uint64_t counters[3]);

/* ---- synthetic inputs (synth.c): DFSG0001 cache of the deterministic R-MAT
 * (kind 0, a = scale) / ER (kind 1, a = n) graph the product's generator
 * builds, for the reference arm.  Returns 0 or a negative code. */
int dor_generate_cache(int kind, uint64_t a, uint64_t m, uint64_t seed, const char *path,
                       uint32_t *n_out);

#ifdef __cplusplus
}
#endif
#endif
