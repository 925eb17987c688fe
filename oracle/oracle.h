/*
 * oracle.h — CPU restatement of the reference (aigsage) hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2511_18297_b200/)
 * links or calls this; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker.
 *
 * Every function restates one reference function; the file:line it follows is
 * cited beside each declaration (paths relative to /root/reference/proj/core).
 * Literals are encoded AIGER-style: lit = 2*node + inverted.
 *
 * Pinning: the restatement is checked against the real reference sources,
 * compiled from /root/reference into oracle/_ref (see oracle/Makefile and
 * oracle/ref_shim.cpp), and against golden fixtures generated from that build
 * (tests/golden/, script tests/golden/make_golden.py). The dense transform of
 * the forward pass (Eigen GEMM, src/gnn.cpp:46-51) cannot be pinned — Eigen is
 * absent — so logits parity at that boundary is "unpinned".
 */
#ifndef GROOT_ORACLE_H
#define GROOT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- circuitgen: src/circuitgen.cpp:13-133 ------------------------------ */
/* Sizes of gen_csa_multiplier(width): inputs 2w, outputs 2w, AND count. */
int orc_csa_sizes(uint32_t width, uint32_t* num_inputs, uint32_t* num_ands,
                  uint32_t* num_outputs);
/* and_lits: 2*num_ands (left,right); out_lits: num_outputs;
 * labels: 1 + num_inputs + num_ands + num_outputs (GroundTruth::labels). */
int orc_gen_csa(uint32_t width, uint32_t* and_lits, uint32_t* out_lits, uint8_t* labels);

/* --- encode: src/encode.cpp:14-68 --------------------------------------- */
/* n = 1 + I + A + O; E = 2A + O; nnz = 2E. */
int orc_encode(uint32_t num_inputs, uint32_t num_ands, const uint32_t* and_lits,
               uint32_t num_outputs, const uint32_t* out_lits,
               uint8_t* features /*4n*/, uint32_t* fwd_edges /*2E*/,
               uint64_t* row_ptr /*n+1*/, uint32_t* col_idx /*2E*/, uint32_t* degree /*n*/);
/* build_symmetric_csr, src/encode.cpp:14-31 */
int orc_build_csr(uint32_t n, uint64_t num_edges, const uint32_t* edges,
                  uint64_t* row_ptr, uint32_t* col_idx);
/* batch, src/encode.cpp:70-101 (copies >= 2; copies == 1 is the identity) */
int orc_batch(uint32_t n, uint64_t num_edges, const uint64_t* row_ptr, const uint32_t* col_idx,
              const uint8_t* features, const uint8_t* labels, const uint32_t* fwd_edges,
              uint32_t copies, uint64_t* o_row_ptr, uint32_t* o_col_idx, uint8_t* o_features,
              uint8_t* o_labels, uint32_t* o_degree, uint32_t* o_fwd_edges);

/* --- partition: src/partition.cpp:301-312, 402-513 ---------------------- */
int orc_topo_chunks(uint32_t n, uint32_t k, uint32_t* part_of);

typedef struct orc_parts orc_parts;
/* build_partitions (regrow when with_boundary, core_subgraphs otherwise). */
orc_parts* orc_regrow(uint32_t n, const uint64_t* row_ptr, const uint32_t* col_idx,
                      uint64_t num_edges, const uint32_t* fwd_edges, const uint32_t* part_of,
                      uint32_t k, int with_boundary);
uint32_t orc_parts_count(const orc_parts* h);
void orc_parts_sizes(const orc_parts* h, uint32_t p, uint32_t* num_core, uint32_t* num_boundary,
                     uint64_t* num_edges);
void orc_parts_copy(const orc_parts* h, uint32_t p, uint32_t* core, uint32_t* boundary,
                    uint32_t* edges /*2*num_edges local ids*/);
void orc_parts_free(orc_parts* h);
double orc_crossing_fraction(uint64_t num_edges, const uint32_t* fwd_edges, const uint32_t* part_of);
uint64_t orc_edge_cut(uint64_t num_edges, const uint32_t* fwd_edges, const uint32_t* part_of);

/* --- spmm: src/spmm.cpp:9-127, inc/spmm.hpp:106-204 ---------------------- */
int orc_degree_sort(uint32_t rows, const uint64_t* row_ptr, uint32_t* perm, uint64_t* sorted_row_ptr);
typedef struct orc_plan orc_plan;
orc_plan* orc_build_plan(uint32_t rows, const uint64_t* row_ptr, uint32_t hd_threshold,
                         uint32_t ld_threshold, uint32_t nz_budget);
/* counts[0..5] = hd_rows, mid_rows, ld_groups, work_units, ld_row_begin, ld_row_end */
void orc_plan_counts(const orc_plan* p, uint64_t counts[6]);
/* hd_rows, mid_rows (sorted-row ids), ld_groups (3 per group), units (6 u64 per unit:
 * kind, sorted_row, row_count, nz_begin, nz_end, partial_slot), perm. Any may be NULL. */
void orc_plan_copy(const orc_plan* p, uint32_t* hd_rows, uint32_t* mid_rows, uint32_t* ld_groups,
                   uint64_t* units, uint32_t* perm);
/* out = m * dense (values given), following execute's accumulation order. */
int orc_plan_execute(const orc_plan* p, uint32_t rows, const uint64_t* row_ptr,
                     const uint32_t* col_idx, const double* values, const double* dense,
                     uint32_t f, double* out);
void orc_plan_free(orc_plan* p);
/* reference_spmm, inc/spmm.hpp:184-195 */
int orc_reference_spmm(uint32_t rows, const uint64_t* row_ptr, const uint32_t* col_idx,
                       const double* values, const double* dense, uint32_t f, double* out);

/* --- gnn: src/gnn.cpp:37-52, 113-178, 259-300, 330-372 ------------------- */
/* Parameter count in ASG1 order (per layer W_self, W_neigh, bias; W_out, b_out). */
uint64_t orc_param_count(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes);
int orc_init_model(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                   uint32_t depth, double* params);
/* logits n x classes (fp64). threads = 0 picks hardware concurrency. */
int orc_forward(uint32_t n, const uint64_t* row_ptr, const uint32_t* col_idx,
                const uint8_t* features, uint32_t depth, uint32_t in_dim, uint32_t hidden,
                uint32_t classes, const double* params, double* logits, unsigned threads);
/* argmax (first max wins) + confusion[truth][pred] + accuracy; score_rows/finish_prediction */
int orc_classify(uint32_t n, uint32_t classes, const double* logits, const uint8_t* truth,
                 uint8_t* pred, uint64_t* confusion, double* accuracy);
/* full-batch Adam training (src/gnn.cpp:180-255); params in/out receive the final weights. */
int orc_train(uint32_t n, const uint64_t* row_ptr, const uint32_t* col_idx,
              const uint8_t* features, const uint8_t* labels, uint32_t epochs, double lr,
              uint64_t seed, double* params /*out, 4-32-32-32-32-5*/, double* final_loss,
              double* final_accuracy);

const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
