/*
 * dippm_host.h — C ABI of the native host front end (libdippm_host.so):
 * graph JSON document -> operator-graph encoding + static features, the
 * step in front of the B200 hot path.
 *
 * Replaces, for a batch of documents and on all host cores:
 *   graph_ir.parse_graph_json   /root/reference/pkg/src/dippm/graph_ir.py:212-297
 *     (validation :180-209, _topological_order :300-323, infer_shapes :357-499)
 *   graph_ir.with_batch_size    graph_ir.py:502-529
 *   featurize.create_graph_encoding  featurize.py:186-190
 *     (operator_graph :106-163, encode_node :166-183)
 *   featurize.static_features   featurize.py:256-267 (compute_macs :204-253)
 * Outputs are bit-identical to the reference (features are float64 computed
 * with the same libm log1p; integer results exact), errors are reported as
 * the reference's exception class per document.
 *
 * Conventions: plain pointers and sizes; host memory only (no CUDA); the
 * result object is opaque and owned by the caller (dippm_feat_free).
 */
#ifndef DIPPM_HOST_H_
#define DIPPM_HOST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DIPPM_HOST_ABI_VERSION 2

/* Per-document status: the reference exception class (errors.py:8-83). */
enum dippm_feat_status {
  DIPPM_FEAT_OK = 0,
  DIPPM_FEAT_MALFORMED_DOCUMENT = 1,
  DIPPM_FEAT_CYCLIC_GRAPH = 2,
  DIPPM_FEAT_DANGLING_REFERENCE = 3,
  DIPPM_FEAT_BAD_SHAPE = 4,
  DIPPM_FEAT_SHAPE_MISMATCH = 5,
  DIPPM_FEAT_UNDERSPECIFIED = 6,
  DIPPM_FEAT_EMPTY_GRAPH = 7,
  DIPPM_FEAT_INVALID_SPEC = 8,
  DIPPM_FEAT_VALUE_ERROR = 9,   /* Python ValueError/IndexError/OverflowError paths (non-DippmError) */
  DIPPM_FEAT_UNSUPPORTED = 10   /* integers beyond int64 (the reference would use big ints) */
};

typedef struct dippm_feat_batch dippm_feat_batch;

int32_t dippm_host_abi_version(void);

/* Featurise `count` documents (UTF-8 JSON, docs[i] of lens[i] bytes).
 * batch_override[i] > 0 applies with_batch_size(graph, batch_override[i]);
 * 0 (or a NULL array) keeps the document's batch; < 0 is InvalidSpec.
 * threads <= 0 uses all hardware threads.  Never returns NULL except on
 * allocation failure. */
dippm_feat_batch* dippm_featurize_docs(const char* const* docs, const int64_t* lens, int64_t count,
                                       const int64_t* batch_override, int32_t threads);

int64_t dippm_feat_count(const dippm_feat_batch* b);
/* status of document i; the message (NUL-terminated, truncated to cap) goes to msg if non-NULL */
int32_t dippm_feat_status(const dippm_feat_batch* b, int64_t i, char* msg, int64_t cap);
/* graph name of document i (copied into buf, NUL-terminated); returns its byte length */
int64_t dippm_feat_name(const dippm_feat_batch* b, int64_t i, char* buf, int64_t cap);
/* num_nodes[i], num_edges[i] of every document (0 for failed documents); returns the totals */
void dippm_feat_sizes(const dippm_feat_batch* b, int64_t* num_nodes, int64_t* num_edges, int64_t* total_nodes,
                      int64_t* total_edges);
/* Concatenated outputs in document order (failed documents contribute nothing):
 *   x       double [total_nodes, 32]  feature rows (featurize.py:166-183)
 *   edges   int64  [total_edges, 2]   (src, dst) positions local to each graph
 *   fs_int  int64  [count, 5]         macs, batch, t_conv, t_dense, t_relu (zeros on failure)
 *   x32     float  [total_nodes, 32]  optional (may be NULL): x rounded to fp32 for the device
 * Any pointer may be NULL to skip that output. */
void dippm_feat_export(const dippm_feat_batch* b, double* x, int64_t* edges, int64_t* fs_int, float* x32);
/* The whole batch in the device layout device.upload_batch / dippm_build_csr_grouped take
 * (what FeaturizedBatch.collate builds in Python), written straight into the caller's
 * (typically pinned) buffers; any pointer may be NULL:
 *   x32       float  [total_nodes, 32]  feature rows rounded to fp32
 *   src, dst  int64  [total_edges]      edge endpoints as batch-global node ids
 *   graph_ptr int32  [count + 1]        node offsets; edge_ptr int64 [count + 1] edge offsets
 *   fs64      double [count, 5]         log1p static features (fs_log, StaticFeatures.as_vector)
 * Failed documents contribute no nodes or edges (callers normally reject the batch first). */
void dippm_feat_collate(const dippm_feat_batch* b, float* x32, int64_t* src, int64_t* dst, int32_t* graph_ptr,
                        int64_t* edge_ptr, double* fs64);
/* Per-document metadata in one call (any pointer may be NULL):
 *   status  int32 [count]      (dippm_feat_status codes)
 *   fs_log  double [count, 5]  StaticFeatures.as_vector = log1p of the five integers (featurize.py:76-87)
 *   name_off int64 [count + 1] and names (UTF-8, concatenated; names_cap bytes available):
 *   returns the total name bytes (call with names = NULL first to size the buffer). */
int64_t dippm_feat_meta(const dippm_feat_batch* b, int32_t* status, double* fs_log, int64_t* name_off, char* names,
                        int64_t names_cap);
void dippm_feat_free(dippm_feat_batch* b);

#ifdef __cplusplus
}
#endif

#endif /* DIPPM_HOST_H_ */
