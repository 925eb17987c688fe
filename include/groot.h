/*
 * groot.h — C ABI of the B200-native GROOT hot path (libgroot_b200.so).
 *
 * The reference (aigsage, /root/reference/proj/core) exposes a C++ operator API
 * (free functions over value types). This header is the drop-in boundary for
 * that path: plain pointers and sizes, no C++ or torch types, int status codes.
 * Each entry point names the reference function it replaces (file:line,
 * relative to /root/reference/proj/core). The C++ mirror of the reference API
 * (include/groot_aigsage.hpp, namespace aigsage) is implemented on top of it.
 *
 * Conventions
 *  - Literals are AIGER-encoded: lit = 2*node + inverted (inc/aig.hpp:13-21).
 *  - Graph, assignment, partition and model objects are opaque handles whose
 *    storage lives in device memory (HBM) of the device current at creation.
 *  - Status: GROOT_OK (0); GROOT_EINVAL (1) where the reference throws
 *    std::invalid_argument; GROOT_ERUNTIME (2) where it throws
 *    std::runtime_error (I/O, format); GROOT_ECUDA (3); GROOT_ENCCL (4).
 *    groot_last_error() returns the message (thread-local) — same text as the
 *    reference's exception where one exists.
 *  - Every call is synchronous with respect to the host unless it is a "_dev"
 *    entry point, which only enqueues work on the library stream
 *    (groot_set_stream) and takes device pointers.
 *  - There is no CPU fallback: without a CUDA device every compute entry point
 *    returns GROOT_ECUDA.
 */
#ifndef GROOT_H
#define GROOT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GROOT_OK 0
#define GROOT_EINVAL 1
#define GROOT_ERUNTIME 2
#define GROOT_ECUDA 3
#define GROOT_ENCCL 4

#define GROOT_NUM_CLASSES 5

typedef struct groot_graph groot_graph;         /* EdaGraph, inc/encode.hpp:18-31 */
typedef struct groot_assignment groot_assignment; /* PartitionAssignment, inc/partition.hpp:14-17 */
typedef struct groot_parts groot_parts;         /* vector<AugmentedPartition>, inc/partition.hpp:23-33 */
typedef struct groot_model groot_model;         /* Model, inc/gnn.hpp:26-33 */

/* ---- library ------------------------------------------------------------ */
const char* groot_last_error(void);
int groot_version(void);
/* Stream for all device work (cudaStream_t passed as void*); NULL = legacy default. */
int groot_set_stream(void* stream);
void* groot_get_stream(void);
int groot_device_synchronize(void);
/* Counter of kernels the library launched since the last reset (bench evidence). */
uint64_t groot_kernel_launches(void);
void groot_reset_kernel_launches(void);
/* Per-kernel CUDA-event timing on the library stream. enable(1) clears and
 * starts recording; read() returns, per kernel name, the summed milliseconds
 * and launch count (names: max entries of 48 chars each). */
int groot_profile_enable(int on);
int groot_profile_read(uint32_t max, char* names, double* total_ms, uint64_t* launches,
                       uint32_t* count);
/* Release cached device blocks held by the library's caching allocator. */
int groot_empty_cache(void);

/* ---- AIG sources (host; input side of the path) --------------------------
 * gen_csa_multiplier (src/circuitgen.cpp:66-133): deterministic CSA array.
 * Two-call pattern: sizes first, then fill caller buffers. labels has
 * n = 1 + num_inputs + num_ands + num_outputs entries (GroundTruth::labels). */
int groot_csa_sizes(uint32_t width, uint32_t* num_inputs, uint32_t* num_ands,
                    uint32_t* num_outputs);
int groot_gen_csa(uint32_t width, uint32_t* and_lits /*2*num_ands*/, uint32_t* out_lits,
                  uint8_t* labels);
/* GroundTruth::supports of gen_csa_multiplier (src/circuitgen.cpp:30-32,
 * 50-62): per adder root (HA sum / carry, FA sum / MAJ root) 5 u32 -- root
 * node, arity (2 or 3), three support literals (third 0 when arity 2).
 * records may be NULL (count only). */
int groot_csa_supports(uint32_t width, uint32_t* count, uint32_t* records);
/* Radix-4 Booth multiplier AIG (BASELINE config 3; no reference generator
 * exists): unsigned width x width -> 2*width product bits,
 * same input/output conventions and label classes as groot_gen_csa; encoder
 * and selector gates labelled AND, adder roots XOR / MAJ. Constants folded. */
int groot_booth_sizes(uint32_t width, uint32_t* num_inputs, uint32_t* num_ands, uint32_t* num_outputs);
int groot_gen_booth(uint32_t width, uint32_t* and_lits /*2*num_ands*/, uint32_t* out_lits, uint8_t* labels);
/* parse_aiger (src/aig.cpp:47-88), ASCII "aag" text, same validation and error
 * texts. Sizes via *_sizes, then groot_aiger_fill. */
int groot_aiger_sizes(const char* text, size_t len, uint32_t* num_inputs, uint32_t* num_ands,
                      uint32_t* num_outputs);
int groot_aiger_fill(const char* text, size_t len, uint32_t* and_lits, uint32_t* out_lits);

/* ---- feature build: encode (src/encode.cpp:33-68) ------------------------
 * AIG (host arrays) -> device-resident EdaGraph: 4-bit node features (K1),
 * fwd_edges, symmetric CSR with per-row ascending col_idx (K2). labels: host
 * array of n entries (may be NULL -> zeros). */
int groot_encode(uint32_t num_inputs, uint32_t num_ands, const uint32_t* and_lits,
                 uint32_t num_outputs, const uint32_t* out_lits, const uint8_t* labels,
                 groot_graph** out);
/* batch (src/encode.cpp:70-101): b disjoint copies, node i of copy k -> k*n+i (K3). */
int groot_batch(const groot_graph* g, uint32_t copies, groot_graph** out);
/* Upload an EdaGraph given as host arrays (row_ptr u64[n+1], col_idx u32[nnz],
 * features u8[4n], labels u8[n], fwd_edges u32[2E]); features/labels/edges may be NULL. */
int groot_graph_from_host(uint32_t n, const uint64_t* row_ptr, const uint32_t* col_idx,
                          const uint8_t* features, const uint8_t* labels, uint64_t num_edges,
                          const uint32_t* fwd_edges, groot_graph** out);
/* build_symmetric_csr (src/encode.cpp:14-31) on the device from a forward edge
 * list: rows ascending, duplicates kept. features/labels may be NULL. */
int groot_graph_from_edges(uint32_t n, const uint8_t* features, const uint8_t* labels, uint64_t num_edges,
                           const uint32_t* fwd_edges, groot_graph** out);
int groot_graph_sizes(const groot_graph* g, uint32_t* n, uint64_t* nnz, uint64_t* num_edges);
/* Copy any subset of the EdaGraph arrays back to host (NULL = skip). */
int groot_graph_copy_out(const groot_graph* g, uint64_t* row_ptr, uint32_t* col_idx,
                         uint8_t* features, uint8_t* labels, uint32_t* degree,
                         uint32_t* fwd_edges);
/* Device pointers of the resident arrays (row_ptr is u32[n+1] on device). */
int groot_graph_device_ptrs(const groot_graph* g, const uint32_t** row_ptr,
                            const uint32_t** col_idx, const uint8_t** features,
                            const uint8_t** labels, const uint32_t** fwd_edges);
void groot_graph_free(groot_graph* g);

/* ---- partition ------------------------------------------------------------
 * partition_topo_chunks (src/partition.cpp:301-312): part p = [n*p/k, n*(p+1)/k). */
int groot_partition_topo_chunks(const groot_graph* g, uint32_t k, groot_assignment** out);
/* partition_multilevel (src/partition.cpp:314-367) replacement: the topo
 * chunks refined on the device by deterministic, size-constrained label
 * propagation (part sizes <= ceil(1.05 n / k), never empty), so it terminates
 * for every k (the reference livelocks for k >= 8 in rebalance, :259-297).
 * Equal to the reference's result where that terminates and its refined-topo
 * candidate wins. seed: accepted for the reference's signature (no random
 * choice is made). rounds / moves (may be NULL): LP rounds run, nodes moved. */
int groot_partition_multilevel(const groot_graph* g, uint32_t k, uint64_t seed, groot_assignment** out,
                               uint32_t* rounds, uint64_t* moves);
/* load_assignment (src/partition.cpp:369-392): "node part" lines, same checks. */
int groot_load_assignment(const char* path, uint32_t n, groot_assignment** out);
/* From a host part_of[n] array (validated like load_assignment). */
int groot_assignment_from_host(uint32_t n, const uint32_t* part_of, groot_assignment** out);
int groot_assignment_info(const groot_assignment* a, uint32_t* n, uint32_t* k);
int groot_assignment_copy_out(const groot_assignment* a, uint32_t* part_of);
void groot_assignment_free(groot_assignment* a);
/* crossing_fraction / edge_cut (src/partition.cpp:468-474, 508-513). */
int groot_crossing_fraction(const groot_graph* g, const groot_assignment* a, double* fraction);
int groot_edge_cut(const groot_graph* g, const groot_assignment* a, uint64_t* cut);

/* ---- edge re-growth ---------------------------------------------------------
 * regrow (with_boundary=1) / core_subgraphs (0) (src/partition.cpp:402-466):
 * core_nodes ascending, boundary_nodes = sorted-unique 1-hop neighbours in
 * other parts, local ids = cores then boundary, local edges in fwd_edges
 * order with crossing edges appended to part(u) then part(v) (K5, K6). */
int groot_regrow(const groot_graph* g, const groot_assignment* a, int with_boundary,
                 groot_parts** out);
int groot_parts_count(const groot_parts* p, uint32_t* k);
int groot_parts_sizes(const groot_parts* p, uint32_t part, uint32_t* num_core,
                      uint32_t* num_boundary, uint64_t* num_edges);
/* core_nodes, boundary_nodes, edges (2*num_edges local ids); NULL = skip. */
int groot_parts_copy_out(const groot_parts* p, uint32_t part, uint32_t* core_nodes,
                         uint32_t* boundary_nodes, uint32_t* edges);
/* footprint_proxy (src/partition.cpp:476-486). */
int groot_footprint_proxy(const groot_parts* p, uint32_t feature_cols, uint32_t hidden_dim,
                          uint64_t* bytes);
/* materialize (src/partition.cpp:488-506): standalone EdaGraph of one part (K7). */
int groot_materialize(const groot_graph* g, const groot_parts* p, uint32_t part,
                      groot_graph** out);
/* The caller's vector<AugmentedPartition> (e.g. the predict(model, g, parts)
 * argument, src/gnn.cpp:280-291) uploaded as it is: per part p the core
 * nodes core_nodes[core_off[p] .. core_off[p+1]), the boundary nodes and the
 * local edge pairs likewise (offsets: k+1 entries each, starting at 0).
 * Validated: global ids < n, local endpoints < the part's size. */
int groot_parts_from_host(uint32_t n, uint32_t k, const uint64_t* core_off, const uint32_t* core_nodes,
                          const uint64_t* bnd_off, const uint32_t* boundary_nodes, const uint64_t* edge_off,
                          const uint32_t* edges, groot_parts** out);
void groot_parts_free(groot_parts* p);

/* ---- model (src/gnn.cpp:113-138, 330-372) ------------------------------------
 * Parameters in ASG1 order: per layer W_self[in x hid], W_neigh[in x hid],
 * bias[hid]; then W_out[hid x classes], b_out[classes]; fp64 row-major. */
uint64_t groot_param_count(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes);
/* init_model: Glorot U(+-sqrt(6/(in+out))) from mt19937_64(seed), zero biases. */
int groot_init_params(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                      uint32_t depth, double* params);
/* Device model (weights pre-split into TF32 hi/lo for the tensor-core layers).
 * Supported shape: in_dim 4, hidden 32, classes <= 8, depth >= 1. */
int groot_model_create(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                       const double* params, groot_model** out);
int groot_model_load(const char* path, groot_model** out);            /* load_model */
int groot_model_save(const groot_model* m, const char* path);         /* save_model */
int groot_model_info(const groot_model* m, uint32_t* depth, uint32_t* in_dim, uint32_t* hidden,
                     uint32_t* classes);
int groot_model_params(const groot_model* m, double* params);
void groot_model_free(groot_model* m);

/* ---- SageContext: make_context (src/gnn.cpp:140-170) --------------------------
 * Everything the forward derives from the graph alone -- the row classifier
 * (HD band of the degree-polarised split), the per-tile gather plan, the HD
 * chunk plan and the activation buffers -- built on the device and cached on
 * the graph handle (every forward entry point builds what is missing on first
 * use; prepare builds it eagerly). release frees it; the next forward rebuilds. */
int groot_graph_prepare(const groot_graph* g);
int groot_graph_release_context(const groot_graph* g);

/* ---- training: train / loss_and_grads (src/gnn.cpp:180-255) --------------------
 * Full-batch training on the resident graph in fp64 on the device: forward with
 * the whole cache, softmax cross entropy averaged over nodes, backward with the
 * transposed mean aggregation (a_mean_t), Adam with bias correction.
 * init_params NULL -> init_model(seed) (Glorot, mt19937_64). params_out gets
 * the trained parameters (ASG1 order); loss_out / accuracy_out (epochs
 * entries each, may be NULL) the per-epoch training loss and accuracy before
 * that epoch's update (TrainStats). Supported: in_dim 4, hidden <= 64,
 * classes <= 8. Throws (GROOT_ERUNTIME) on a non-finite loss. */
int groot_train(const groot_graph* g, uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                uint32_t epochs, double learning_rate, uint64_t seed, double beta1, double beta2, double adam_eps,
                const double* init_params, double* params_out, double* loss_out, double* accuracy_out);
/* loss_and_grads (src/gnn.cpp:180-209): mean loss and its gradient (ASG1 order). */
int groot_loss_and_grads(const groot_graph* g, uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                         const double* params, double* grads_out, double* loss);

/* ---- layer forward + classify ------------------------------------------------
 * forward (src/gnn.cpp:172-178): logits n x classes, fp32 on device (written to
 * host buffer logits_host). */
int groot_forward(const groot_model* m, const groot_graph* g, float* logits_host);
/* predict_full (src/gnn.cpp:293-300): labels u8[n] (argmax, first max wins),
 * confusion[truth*5+pred] (u64[25]) and accuracy; any output may be NULL. */
int groot_predict_full(const groot_model* m, const groot_graph* g, uint8_t* labels_host,
                       uint64_t* confusion, double* accuracy);
/* predict (src/gnn.cpp:280-291): every part's augmented subgraph forwarded,
 * each node scored from the part that owns it as a core node. */
int groot_predict(const groot_model* m, const groot_graph* g, const groot_parts* p,
                  uint8_t* labels_host, uint64_t* confusion, double* accuracy);

/* predict restricted to the parts in part_ids (multi-GPU: each rank forwards
 * its own parts): labels_host (n entries, in/out) receives the classes of the
 * core nodes of those parts; all other entries are left unchanged. */
int groot_predict_parts(const groot_model* m, const groot_graph* g, const groot_parts* p,
                        const uint32_t* part_ids, uint32_t count, uint8_t* labels_host);

/* Device-resident session entry points (no host copies; work enqueued on the
 * library stream). labels_dev u8[n], logits_dev f32[n*classes] (NULL = skip),
 * confusion_dev u64[25] (NULL = skip; accumulated, caller zeroes). */
int groot_predict_full_dev(const groot_model* m, const groot_graph* g, uint8_t* labels_dev,
                           float* logits_dev, uint64_t* confusion_dev);

/* One layer of run_forward (src/gnn.cpp:37-52) on a resident graph, device
 * buffers, enqueued on the library stream (the building block of the
 * exact-halo multi-GPU mode, paper_2511_18297_b200/shard.py):
 *   layer 0: node features -> hout (n x hidden);  0 < layer < depth-1: hin -> hout;
 *   layer depth-1: hin -> head + first-max argmax -> labels_dev (u8[n]), logits_dev
 *   (n x classes, may be NULL). Every row is computed from its own neighbour list. */
int groot_layer_dev(const groot_model* m, const groot_graph* g, uint32_t layer, const float* hin_dev,
                    float* hout_dev, uint8_t* labels_dev, float* logits_dev);
/* End-to-end from AIG host arrays: encode -> batch -> predict_full, classes to
 * host (the drop-in for run_cell's encode/batch/predict chain). */
int groot_classify_aig(const groot_model* m, uint32_t num_inputs, uint32_t num_ands,
                       const uint32_t* and_lits, uint32_t num_outputs, const uint32_t* out_lits,
                       const uint8_t* labels, uint32_t copies, uint8_t* labels_out,
                       uint64_t* confusion, double* accuracy);

/* Differential-test path: the same forward with thread-per-row CUDA kernels
 * (no tensor cores, no HD/LD split). Not used by the product entry points. */
int groot_debug_forward_naive(const groot_model* m, const groot_graph* g, float* logits_host,
                              uint8_t* labels_host);

/* ---- verification consumer of the classes (src/verify.cpp:220-418) -----------
 * backward_rewrite: label-guided backward rewriting of a width-bit multiplier
 * candidate's output word polynomial against (sum 2^i a_i)(sum 2^j b_j);
 * labels (num_labels >= 1 + ni + na, classes as NodeClass) steer XOR / MAJ
 * substitutions, each validated on its cone's truth table first, so wrong
 * labels cost time, never soundness. support_off (num_nodes+1) / support_nodes
 * give per-node supports (node ids; both may be NULL). monomial_cap 0 = the
 * reference's 2,000,000. Outputs (any may be NULL): equivalent, inconclusive
 * (cap hit), residual term count, counts[3] = {substitutions, shortcuts,
 * fallbacks}. groot_backward_rewrite_residual(): the residual as text (first
 * 64 terms, "coeff*x3*x9 + ..."; thread-local, valid until the next call). */
int groot_backward_rewrite(uint32_t num_inputs, uint32_t num_ands, const uint32_t* and_lits, uint32_t num_outputs,
                           const uint32_t* out_lits, const uint8_t* labels, uint32_t num_labels,
                           const uint32_t* support_off, const uint32_t* support_nodes, uint32_t width,
                           uint64_t monomial_cap, int32_t* equivalent, int32_t* inconclusive,
                           uint64_t* residual_terms, uint64_t* counts);
const char* groot_backward_rewrite_residual(void);
/* truth_table_equiv (src/verify.cpp:398-416): exhaustive simulation against
 * the integer product, 2*width <= 20. */
int groot_truth_table_equiv(uint32_t num_inputs, uint32_t num_ands, const uint32_t* and_lits, uint32_t num_outputs,
                            const uint32_t* out_lits, uint32_t width, int32_t* equivalent);
/* simulate (src/aig.cpp:115-138): output bits for one input assignment. */
int groot_simulate(uint32_t num_inputs, uint32_t num_ands, const uint32_t* and_lits, uint32_t num_outputs,
                   const uint32_t* out_lits, const uint8_t* inputs, uint8_t* outputs);

/* ---- degree-polarised aggregation (src/spmm.cpp, inc/spmm.hpp) ---------------
 * build_plan (src/spmm.cpp:37-127) row classifier on device: per-band counts
 * and the reference plan arrays. counts[6] = {hd_rows, mid_rows, ld_groups,
 * work_units, ld_row_begin, ld_row_end}; arrays may be NULL. units: 6 u64 per
 * unit {kind(0 HD,1 LD,2 MID), sorted_row, row_count, nz_begin, nz_end, slot}. */
int groot_build_plan(const groot_graph* g, uint32_t hd_threshold, uint32_t ld_threshold,
                     uint32_t nz_budget, uint64_t* counts, uint32_t* perm, uint32_t* hd_rows,
                     uint32_t* mid_rows, uint32_t* ld_groups, uint64_t* units);
/* out = D^-1 A * dense (mean aggregation, spmm::execute with a_mean values),
 * dense/out f32 row-major on host, f in {4, 32} or any f <= 256. */
int groot_spmm_mean(const groot_graph* g, const float* dense, uint32_t f, float* out);
/* spmm::execute over a host CsrMatrix<float> / CsrMatrix<double>
 * (inc/spmm.hpp:106-181) on the device: nonzeros accumulated in order with
 * separately rounded multiply and add; rows of degree >= hd_threshold summed
 * as 32 chunk partials added in ascending order, as the HD band of a plan
 * built with that threshold -- so the result is bitwise the reference's
 * execute. hd_threshold 0: the plain row loop (reference_spmm,
 * inc/spmm.hpp:183-195). values NULL -> 1/deg (a_mean). */
int groot_spmm_csr(uint32_t rows, uint32_t cols, const uint64_t* row_ptr, const uint32_t* col_idx,
                   const float* values, const float* dense, uint32_t f, uint32_t hd_threshold, float* out);
int groot_spmm_csr_f64(uint32_t rows, uint32_t cols, const uint64_t* row_ptr, const uint32_t* col_idx,
                       const double* values, const double* dense, uint32_t f, uint32_t hd_threshold, double* out);
/* build_plan over a host row_ptr (build_plan(rows, span row_ptr, ...),
 * src/spmm.cpp:37-127), same outputs as groot_build_plan. */
int groot_build_plan_rows(uint32_t rows, const uint64_t* row_ptr, uint32_t hd_threshold, uint32_t ld_threshold,
                          uint32_t nz_budget, uint64_t* counts, uint32_t* perm, uint32_t* hd_rows,
                          uint32_t* mid_rows, uint32_t* ld_groups, uint64_t* units);
/* degree_sort (src/spmm.cpp:9-35): stable ascending-by-degree permutation
 * (perm[sorted] = original row) and the row pointers in that order (rows+1). */
int groot_degree_sort(uint32_t rows, const uint64_t* row_ptr, uint32_t* perm, uint64_t* sorted_row_ptr);
/* Device variant of the mean SpMM (bench / roofline): pointers on device. */
int groot_spmm_mean_dev(const groot_graph* g, const float* dense_dev, uint32_t f, float* out_dev);

#ifdef __cplusplus
}
#endif
#endif /* GROOT_H */
