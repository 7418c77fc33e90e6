// The whole w-product (algebra.py:43-51) as ONE C-ABI call: K1 on a, K1 on b,
// one K3 over all p wavelet slices, K2 -- the four launches of
// inverse_w(face_product(forward_w(a), forward_w(b))) without a round trip
// through Python between them.  A call that repeats the previous call's
// arguments exactly (same pointers, shapes, levels and stream: a user looping
// over resident tensors, the config-1 benchmark) replays a CUDA graph of the
// four launches captured on the second occurrence; anything else runs them
// eagerly.  Results are identical either way (same kernels, same arguments).
#include <string.h>

#include <mutex>

#include "wt_common.cuh"

namespace {

struct Key {
  const double *a, *b;
  double *c;
  void* ws;
  int64_t n1, n2, n3, p;
  int levels;
  void* stream;
  int device;
  bool operator==(const Key& o) const { return memcmp(this, &o, sizeof(Key)) == 0; }
};

struct Cached {
  Key key;
  int seen = 0;  // consecutive calls with this key
  cudaGraphExec_t exec = nullptr;
};

thread_local Cached g_last{};  // per host thread (streams are per thread in practice)

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

int run_eager(const Key& k) {
  const int64_t s1 = k.p * k.n1 * k.n2, s2 = k.p * k.n2 * k.n3;
  double* pa = static_cast<double*>(k.ws);
  double* pb = reinterpret_cast<double*>(static_cast<char*>(k.ws) + align256(sizeof(double) * s1));
  double* pc = reinterpret_cast<double*>(reinterpret_cast<char*>(pb) + align256(sizeof(double) * s2));
  if (int e = wt_lift_fwd_f64(k.a, k.n1, k.n2, k.p, k.levels, pa, WT_LAYOUT_SLICE_MAJOR, 0, WT_MASK_ALL, k.stream))
    return e;
  if (int e = wt_lift_fwd_f64(k.b, k.n2, k.n3, k.p, k.levels, pb, WT_LAYOUT_SLICE_MAJOR, 0, WT_MASK_ALL, k.stream))
    return e;
  if (int e = wt_gemm_f64(0, 0, k.n1, k.n3, k.n2, 1.0, pa, k.n2, k.n1 * k.n2, pb, k.n3, k.n2 * k.n3, 0.0, pc, k.n3,
                          k.n1 * k.n3, k.p, k.stream))
    return e;
  return wt_lift_inv_f64(pc, k.n1, k.n3, k.p, k.levels, WT_LAYOUT_SLICE_MAJOR, 0, WT_MASK_ALL, k.c, k.stream);
}

}  // namespace

extern "C" size_t wt_w_product_workspace_bytes(int64_t n1, int64_t n2, int64_t n3, int64_t p) {
  if (n1 < 0 || n2 < 0 || n3 < 0 || p < 0) return 0;
  return align256(sizeof(double) * (size_t)(p * n1 * n2)) + align256(sizeof(double) * (size_t)(p * n2 * n3)) +
         align256(sizeof(double) * (size_t)(p * n1 * n3));
}

extern "C" int wt_w_product_f64(const double* a, const double* b, int64_t n1, int64_t n2, int64_t n3, int64_t p,
                                int levels, double* c, void* workspace, size_t workspace_bytes, void* stream) {
  WT_REQUIRE(n1 >= 1 && n2 >= 1 && n3 >= 1 && p >= 1, "w_product: empty operand");
  WT_REQUIRE(levels >= 1 && p % ((int64_t)1 << levels) == 0, "w_product: 2^%d does not divide %lld", levels,
             (long long)p);
  WT_REQUIRE(a && b && c && workspace, "w_product: null pointer");
  WT_REQUIRE(workspace_bytes >= wt_w_product_workspace_bytes(n1, n2, n3, p), "w_product: workspace too small");
  Key k{};
  k.a = a; k.b = b; k.c = c; k.ws = workspace;
  k.n1 = n1; k.n2 = n2; k.n3 = n3; k.p = p; k.levels = levels; k.stream = stream;
  WT_CUDA(cudaGetDevice(&k.device));
  Cached& g = g_last;
  if (!(g.key == k)) {  // new arguments: eager, remember them
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    g.key = k;
    g.seen = 1;
    return run_eager(k);
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (!g.exec) {
    if (++g.seen < 2) return run_eager(k);
    // second identical call: capture the four launches on a private stream (the
    // caller's may be the legacy default stream, which cannot be captured); the
    // graph is then launched on the caller's stream
    static thread_local cudaStream_t cap = nullptr;
    if (!cap) WT_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    Key kc = k;
    kc.stream = cap;
    cudaGraph_t graph = nullptr;
    WT_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int e = run_eager(kc);
    const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    if (e || ce != cudaSuccess || graph == nullptr) {
      if (graph) cudaGraphDestroy(graph);
      (void)cudaGetLastError();
      g.seen = 0;  // do not retry capturing this key
      return e ? e : run_eager(k);
    }
    const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      g.exec = nullptr;
      (void)cudaGetLastError();
      return run_eager(k);
    }
  }
  WT_CUDA(cudaGraphLaunch(g.exec, st));
  return WT_OK;
}
