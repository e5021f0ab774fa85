// labels.cu — the landmark label store as an opaque handle (§8(a) A10 and
// the §8(b) boundary calls cbfs_labels_*): build it from clusters with one
// cbfs_run (records = Delta + S_v[0..d-1], R14), query it
// (P:1013-1021), and move it between ranks as one flat byte
// image (export / import: the unit the NCCL all-gather of A12 moves).
//
// The store's word size w (Tables 4/8: w = 64, 32, 16, 8) is the
// width of one bit-subset: clusters hold at most w sources, and a record
// (c, v) is Delta (dist_bytes) + d words of w/8 bytes — 17 B at w = 64, d = 2
// (u8 Delta), 3 B at w = 8.  The traversal itself always runs on 64-bit
// subsets; its output writes store the low w bits (all that a cluster of
// <= w sources can set).
//
// Image layout (one device allocation, the handle's own storage):
//   [0, 64)            header {magic "CBFSLBL1", version 2, n, C, d, planes,
//                      dist_bytes, total bytes, word_bits}
//   sizes  [C]         u8 cluster sizes            (padded to 16 bytes)
//   dist   [n][C]      Delta, dist_bytes each       (padded to 16 bytes)
//   masks  [planes][n][C] w-bit bit-subsets S_v[0..planes-1]
#include <cstring>
#include <vector>

#include "common.cuh"

namespace cbfs {

struct LabelHeader {
  char magic[8];
  uint32_t version, n, C, d, planes, dist_bytes;
  uint64_t bytes;
  uint32_t word_bits;
  uint8_t pad[64 - 8 - 6 * 4 - 8 - 4];
};
static_assert(sizeof(LabelHeader) == 64, "64-byte header");

struct Labels {
  int device = 0;
  LabelHeader h{};
  uint8_t* blob = nullptr;  // device image
  uint8_t* sizes() const { return blob + 64; }
  void* dist() const { return blob + 64 + pad16(h.C); }
  void* masks() const { return blob + 64 + pad16(h.C) + pad16((uint64_t)h.n * h.C * h.dist_bytes); }
  static uint64_t pad16(uint64_t x) { return (x + 15) & ~15ull; }
};

static uint64_t image_bytes(uint32_t n, uint32_t C, uint32_t planes, uint32_t dist_bytes, uint32_t word_bits) {
  return 64 + Labels::pad16(C) + Labels::pad16((uint64_t)n * C * dist_bytes) + (uint64_t)planes * n * C * (word_bits / 8);
}

// w = 0: plain landmarks (the paper's "Plain" LL): d = 0 and
// single-source clusters, records are Delta alone (no subset planes)
static bool word_ok(uint32_t w) { return w == 0 || w == 8 || w == 16 || w == 32 || w == 64; }

static void make_header(LabelHeader& h, uint32_t n, uint32_t C, uint32_t d, uint32_t dist_bytes, uint32_t word_bits) {
  std::memset(&h, 0, sizeof h);
  std::memcpy(h.magic, "CBFSLBL1", 8);
  h.version = 2;
  h.word_bits = word_bits;
  h.n = n;
  h.C = C;
  h.d = d;
  h.planes = word_bits == 0 ? 0 : (d > 0 ? d : 1);
  h.dist_bytes = dist_bytes;
  h.bytes = image_bytes(n, C, h.planes, dist_bytes, word_bits);
}

}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_labels_build_w(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters,
                        uint32_t d, uint32_t dist_bytes, uint32_t word_bits, cbfs_labels** out, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  if (!out) return fail(CBFS_EINVAL, "null out");
  *out = nullptr;
  if (!g) return fail(CBFS_EINVAL, "null graph");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (d > CBFS_MAX_D) return fail(CBFS_EUNSUPPORTED, "d > CBFS_MAX_D");
  if (!word_ok(word_bits)) return fail(CBFS_EINVAL, "word_bits must be 0, 8, 16, 32 or 64");
  if (word_bits == 0 && d != 0) return fail(CBFS_EINVAL, "plain landmarks (word_bits 0) need d = 0");
  if (n_clusters && !sizes) return fail(CBFS_EINVAL, "null sizes");
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (word_bits < 64 && n_clusters) {  // a cluster must fit one w-bit word
    std::vector<uint8_t> hs(n_clusters);
    CBFS_CUDA(cudaMemcpyAsync(hs.data(), sizes, n_clusters, cudaMemcpyDefault, st));
    CBFS_CUDA(cudaStreamSynchronize(st));
    for (uint8_t x : hs)
      if (x > (word_bits ? word_bits : 1u)) return fail(CBFS_EINVAL, "a cluster has more sources than the word has bits");
  }
  Labels* L = new Labels();
  L->device = g->device;
  make_header(L->h, g->n, n_clusters, d, dist_bytes, word_bits);
  if (cudaMalloc(&L->blob, L->h.bytes) != cudaSuccess) {
    delete L;
    cudaGetLastError();
    return fail(CBFS_ENOMEM, "label store allocation");
  }
  int rc = CBFS_OK;
  if (cudaMemcpyAsync(L->blob, &L->h, sizeof(LabelHeader), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      (n_clusters && cudaMemcpyAsync(L->sizes(), sizes, n_clusters, cudaMemcpyDefault, st) != cudaSuccess))
    rc = cuda_fail(cudaGetLastError(), "label header");
  if (rc == CBFS_OK && n_clusters)
    rc = run_arrays(g, sources, sizes, n_clusters, d, dist_bytes, L->dist(), word_bits ? L->masks() : nullptr,
                    word_bits ? word_bits / 8 : 8, word_bits ? L->h.planes : 1, nullptr, CBFS_DIR_AUTO, st);
  if (rc == CBFS_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "label build");
  if (rc != CBFS_OK) {
    cudaFree(L->blob);
    delete L;
    return rc;
  }
  *out = reinterpret_cast<cbfs_labels*>(L);
  return CBFS_OK;
}

int cbfs_labels_build(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                      uint32_t dist_bytes, cbfs_labels** out, cbfs_stream stream) {
  return cbfs_labels_build_w(gh, sources, sizes, n_clusters, d, dist_bytes, 64, out, stream);
}

int cbfs_labels_word_bits(const cbfs_labels* lh, uint32_t* word_bits) {
  const Labels* L = reinterpret_cast<const Labels*>(lh);
  if (!L || !word_bits) return fail(CBFS_EINVAL, "null argument");
  *word_bits = L->h.word_bits;
  return CBFS_OK;
}

int cbfs_labels_info(const cbfs_labels* lh, uint32_t* n, uint32_t* n_clusters, uint32_t* d, uint32_t* dist_bytes,
                     uint64_t* image_bytes_out) {
  const Labels* L = reinterpret_cast<const Labels*>(lh);
  if (!L) return fail(CBFS_EINVAL, "null labels");
  if (n) *n = L->h.n;
  if (n_clusters) *n_clusters = L->h.C;
  if (d) *d = L->h.d;
  if (dist_bytes) *dist_bytes = L->h.dist_bytes;
  if (image_bytes_out) *image_bytes_out = L->h.bytes;
  return CBFS_OK;
}

int cbfs_labels_export(const cbfs_labels* lh, void* buf, uint64_t bytes) {
  const Labels* L = reinterpret_cast<const Labels*>(lh);
  if (!L || !buf) return fail(CBFS_EINVAL, "null argument");
  if (bytes < L->h.bytes) return fail(CBFS_EINVAL, "buffer smaller than the label image");
  CBFS_CUDA(cudaSetDevice(L->device));
  CBFS_CUDA(cudaMemcpy(buf, L->blob, L->h.bytes, cudaMemcpyDefault));
  return CBFS_OK;
}

int cbfs_labels_import(cbfs_graph* gh, const void* buf, uint64_t bytes, cbfs_labels** out) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  if (!out) return fail(CBFS_EINVAL, "null out");
  *out = nullptr;
  if (!g || !buf) return fail(CBFS_EINVAL, "null argument");
  if (bytes < sizeof(LabelHeader)) return fail(CBFS_EINVAL, "image too small");
  CBFS_CUDA(cudaSetDevice(g->device));
  LabelHeader h;
  CBFS_CUDA(cudaMemcpy(&h, buf, sizeof h, cudaMemcpyDefault));
  if (std::memcmp(h.magic, "CBFSLBL1", 8) != 0 || h.version != 2) return fail(CBFS_EINVAL, "not a label image");
  if (h.n != g->n) return fail(CBFS_EINVAL, "label image is for another graph size");
  if ((h.dist_bytes != 1 && h.dist_bytes != 2) || h.d > CBFS_MAX_D || h.planes != (h.word_bits == 0 ? 0 : (h.d > 0 ? h.d : 1)) ||
      (h.word_bits == 0 && h.d != 0) ||
      !word_ok(h.word_bits) || h.bytes != image_bytes(h.n, h.C, h.planes, h.dist_bytes, h.word_bits) ||
      bytes < h.bytes)
    return fail(CBFS_EINVAL, "corrupt label image header");
  Labels* L = new Labels();
  L->device = g->device;
  L->h = h;
  if (cudaMalloc(&L->blob, h.bytes) != cudaSuccess) {
    delete L;
    cudaGetLastError();
    return fail(CBFS_ENOMEM, "label store allocation");
  }
  if (cudaMemcpy(L->blob, buf, h.bytes, cudaMemcpyDefault) != cudaSuccess) {
    int rc = cuda_fail(cudaGetLastError(), "label import");
    cudaFree(L->blob);
    delete L;
    return rc;
  }
  *out = reinterpret_cast<cbfs_labels*>(L);
  return CBFS_OK;
}

int cbfs_labels_query(const cbfs_labels* lh, const uint32_t* s, const uint32_t* t, uint64_t q, int32_t* inout_best,
                      cbfs_stream stream) {
  const Labels* L = reinterpret_cast<const Labels*>(lh);
  if (!L) return fail(CBFS_EINVAL, "null labels");
  if (L->h.C == 0) return q && (!s || !t || !inout_best) ? fail(CBFS_EINVAL, "null query arrays") : CBFS_OK;
  CBFS_CUDA(cudaSetDevice(L->device));
  const uint32_t mb = L->h.word_bits ? L->h.word_bits / 8 : 8;
  return query_store(L->h.n, L->h.C, L->h.d, L->h.planes, L->dist(), L->h.dist_bytes, L->masks(), mb, L->sizes(), s, t,
                     q, inout_best, (cudaStream_t)stream);
}

int cbfs_labels_destroy(cbfs_labels* lh) {
  Labels* L = reinterpret_cast<Labels*>(lh);
  if (!L) return CBFS_OK;
  cudaSetDevice(L->device);
  cudaFree(L->blob);
  delete L;
  return CBFS_OK;
}

// Index budget: a (cluster, vertex) record is
// Delta (dist_bytes) plus d bit-subsets of w bits (S_v[0..d-1], R14; d = 0
// keeps S_v[0]); w = 0 is a plain landmark, Delta alone.
int cbfs_record_bytes(uint32_t word_bits, uint32_t d, uint32_t dist_bytes, uint64_t* out_bytes) {
  if (!out_bytes) return fail(CBFS_EINVAL, "null out_bytes");
  if (word_bits != 0 && word_bits != 8 && word_bits != 16 && word_bits != 32 && word_bits != 64)
    return fail(CBFS_EINVAL, "word_bits must be 0, 8, 16, 32 or 64");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (d > CBFS_MAX_D) return fail(CBFS_EUNSUPPORTED, "d > CBFS_MAX_D");
  *out_bytes = dist_bytes + (word_bits ? (uint64_t)(d > 0 ? d : 1) * (word_bits / 8) : 0);
  return CBFS_OK;
}

int cbfs_budget_clusters(uint64_t t_bytes, uint32_t word_bits, uint32_t d, uint32_t dist_bytes, uint64_t* out_r) {
  if (!out_r) return fail(CBFS_EINVAL, "null out_r");
  uint64_t rb = 0;
  int rc = cbfs_record_bytes(word_bits, d, dist_bytes, &rb);
  if (rc) return rc;
  *out_r = t_bytes / rb;
  return CBFS_OK;
}

}  // extern "C"
