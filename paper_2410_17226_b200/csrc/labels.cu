// labels.cu — the landmark label store as an opaque handle (§8(a) A10 and
// the §8(b) boundary calls cbfs_labels_*): build it from clusters with one
// cbfs_run (records = Delta + S_v[0..d-1], R14), query it
// (P:1013-1021), and move it between ranks as one flat byte
// image (export / import: the unit the NCCL all-gather of A12 moves).
//
// Image layout (one device allocation, the handle's own storage):
//   [0, 64)            header {magic "CBFSLBL1", version, n, C, d, planes,
//                      dist_bytes, total bytes}
//   sizes  [C]         u8 cluster sizes            (padded to 16 bytes)
//   dist   [n][C]      Delta, dist_bytes each       (padded to 16 bytes)
//   masks  [planes][n][C] u64 bit-subsets S_v[0..planes-1]
#include <cstring>

#include "common.cuh"

namespace cbfs {

struct LabelHeader {
  char magic[8];
  uint32_t version, n, C, d, planes, dist_bytes;
  uint64_t bytes;
  uint8_t pad[64 - 8 - 6 * 4 - 8];
};
static_assert(sizeof(LabelHeader) == 64, "64-byte header");

struct Labels {
  int device = 0;
  LabelHeader h{};
  uint8_t* blob = nullptr;  // device image
  uint8_t* sizes() const { return blob + 64; }
  void* dist() const { return blob + 64 + pad16(h.C); }
  uint64_t* masks() const {
    return reinterpret_cast<uint64_t*>(blob + 64 + pad16(h.C) + pad16((uint64_t)h.n * h.C * h.dist_bytes));
  }
  static uint64_t pad16(uint64_t x) { return (x + 15) & ~15ull; }
};

static uint64_t image_bytes(uint32_t n, uint32_t C, uint32_t planes, uint32_t dist_bytes) {
  return 64 + Labels::pad16(C) + Labels::pad16((uint64_t)n * C * dist_bytes) + (uint64_t)planes * n * C * 8;
}

static void make_header(LabelHeader& h, uint32_t n, uint32_t C, uint32_t d, uint32_t dist_bytes) {
  std::memset(&h, 0, sizeof h);
  std::memcpy(h.magic, "CBFSLBL1", 8);
  h.version = 1;
  h.n = n;
  h.C = C;
  h.d = d;
  h.planes = d > 0 ? d : 1;
  h.dist_bytes = dist_bytes;
  h.bytes = image_bytes(n, C, h.planes, dist_bytes);
}

}  // namespace cbfs

using namespace cbfs;

extern "C" {

int cbfs_labels_build(cbfs_graph* gh, const uint32_t* sources, const uint8_t* sizes, uint32_t n_clusters, uint32_t d,
                      uint32_t dist_bytes, cbfs_labels** out, cbfs_stream stream) {
  Graph* g = reinterpret_cast<Graph*>(gh);
  if (!out) return fail(CBFS_EINVAL, "null out");
  *out = nullptr;
  if (!g) return fail(CBFS_EINVAL, "null graph");
  if (dist_bytes != 1 && dist_bytes != 2) return fail(CBFS_EINVAL, "dist_bytes must be 1 or 2");
  if (d > CBFS_MAX_D) return fail(CBFS_EUNSUPPORTED, "d > CBFS_MAX_D");
  CBFS_CUDA(cudaSetDevice(g->device));
  cudaStream_t st = (cudaStream_t)stream;
  Labels* L = new Labels();
  L->device = g->device;
  make_header(L->h, g->n, n_clusters, d, dist_bytes);
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
    rc = cbfs_run(gh, sources, sizes, n_clusters, d, dist_bytes, L->dist(), L->masks(), L->h.planes, nullptr,
                  CBFS_DIR_AUTO, stream);
  if (rc == CBFS_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "label build");
  if (rc != CBFS_OK) {
    cudaFree(L->blob);
    delete L;
    return rc;
  }
  *out = reinterpret_cast<cbfs_labels*>(L);
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
  if (std::memcmp(h.magic, "CBFSLBL1", 8) != 0 || h.version != 1) return fail(CBFS_EINVAL, "not a label image");
  if (h.n != g->n) return fail(CBFS_EINVAL, "label image is for another graph size");
  if ((h.dist_bytes != 1 && h.dist_bytes != 2) || h.d > CBFS_MAX_D || h.planes != (h.d > 0 ? h.d : 1) ||
      h.bytes != image_bytes(h.n, h.C, h.planes, h.dist_bytes) || bytes < h.bytes)
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
  return cbfs_query_distance(L->h.n, L->h.C, L->h.d, L->h.planes, L->dist(), L->h.dist_bytes, L->masks(), L->sizes(),
                             s, t, q, inout_best, stream);
}

int cbfs_labels_destroy(cbfs_labels* lh) {
  Labels* L = reinterpret_cast<Labels*>(lh);
  if (!L) return CBFS_OK;
  cudaSetDevice(L->device);
  cudaFree(L->blob);
  delete L;
  return CBFS_OK;
}

}  // extern "C"
