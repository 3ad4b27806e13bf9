// Multi-GPU sharded solve — one rank per GPU, exchanges over NCCL (NVLink /
// NVSwitch), every exchange stream-ordered (no host synchronisation inside a solve).
// Included at the end of capi.cu (uses its context, plan and factor helpers).
//
// Mode groups:
//   head H = modes [0, h): the super-mode sharded in layout L_1 (rank q owns head super-indices
//            [sH_q, sH_q + mH_q)); h = 1 (contiguous blocks of mode 1) or, when every extent is 2,
//            h = log2 P (one head super-index per rank: the first log2 P binary modes);
//   tail G = modes [N - g, N): sharded in layout L_N the same way (g = 1, or log2 P binary modes);
//   pipe K = modes [N - gp, N): the triangular solve's pipeline blocks (gp = 1: contiguous blocks
//            of mode N; binary: one super-index of the last gp modes per block).
// Solve (B in L_N, X returned in L_N):
//   1. forward modes outside G (local in L_N);       2. all-to-all L_N -> L_1 (one grouped P2P);
//   3. forward modes of G (local in L_1);            4. triangular solve pipelined over
//      (rank, block k): block k of rank q needs the head couplings
//        C_q[k] -= T_H[q rows, q' cols] x_H Y_q'[k]  from every q' > q with a nonzero block
//      (T_H = the Kronecker sum of the head modes' T_j: T_1 for h = 1, hypercube neighbours for
//      binary heads), received point-to-point, then solves locally with the head / pipe blocks'
//      diagonal parts (extent-1 modes folded into the denominator), sends Y_q[k] to the lower
//      ranks and applies the pipe couplings C_q[k'' < k] -= T_K[k'' rows, k cols] x_K Y_q[k];
//   5. inverse modes outside H (local in L_1);       6. all-to-all L_1 -> L_N;
//   7. inverse modes of H (local in L_N).
// All P2P traffic of a rank goes through one communication stream in program order (send(k) to
// the lower ranks and recv(k - 1) from the higher ranks form one group), with events handing
// buffers between it and the compute stream, so sends overlap the pipe updates and the next
// block; received blocks are double-buffered by block parity.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>

namespace {

// NCCL is opened at run time (the copy torch already loaded when present): no link-time
// dependency and no second NCCL in a torch process.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::decay_t<decltype(fp)>>(dlsym(h, name));
      if (!fp && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  if (!api.error.empty()) throw Error(NDS_ERR_OTHER, api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(NDS_ERR_OTHER, std::string("NCCL ") + what + ": " + nccl_api().error_string(r));
}

}  // namespace

// Point-to-point transport of one rank: NCCL, or an in-process loopback between ranks that share
// one device (tests: P ranks as host threads of one process).
struct nds_comm {
  int rank = 0, world = 1;
  virtual ~nds_comm() = default;
  virtual void group_begin() = 0;
  virtual void group_end() = 0;
  virtual void send(const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
};

namespace {

struct NcclComm final : nds_comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl_api().comm_destroy(comm);
  }
  void group_begin() override { nccl_check(nccl_api().group_start(), "group start"); }
  void group_end() override { nccl_check(nccl_api().group_end(), "group end"); }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
    nccl_check(nccl_api().send(buf, bytes, ncclUint8, peer, comm, s), "send");
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
    nccl_check(nccl_api().recv(buf, bytes, ncclUint8, peer, comm, s), "recv");
  }
};

// Loopback: a send posts {pointer, ready event} to the (src, dst) mailbox; the receiver's stream
// waits for the event and copies; the sender's stream then waits for the copy. Within a group all
// sends are posted before any receive is served (so an all-to-all cannot deadlock), like NCCL.
struct LoopHub {
  struct Msg {
    const void* ptr;
    size_t bytes;
    cudaEvent_t ready, done;
    bool taken = false;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> box;
};

struct LoopComm final : nds_comm {
  std::shared_ptr<LoopHub> hub;
  int depth = 0;
  struct Send {
    std::shared_ptr<LoopHub::Msg> m;
    cudaStream_t s;
  };
  struct Recv {
    void* buf;
    size_t bytes;
    int peer;
    cudaStream_t s;
  };
  std::vector<Send> sends;
  std::vector<Recv> recvs;
  void group_begin() override { ++depth; }
  void group_end() override {
    if (--depth == 0) flush();
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
    auto m = std::make_shared<LoopHub::Msg>();
    m->ptr = buf;
    m->bytes = bytes;
    NDS_CUDA(cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming));
    NDS_CUDA(cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming));
    NDS_CUDA(cudaEventRecord(m->ready, s));
    {
      std::lock_guard<std::mutex> lk(hub->mu);
      hub->box[{rank, peer}].push_back(m);
    }
    hub->cv.notify_all();
    sends.push_back({m, s});
    if (depth == 0) flush();
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
    recvs.push_back({buf, bytes, peer, s});
    if (depth == 0) flush();
  }
  void flush() {
    for (const Recv& r : recvs) {
      std::shared_ptr<LoopHub::Msg> m;
      {
        std::unique_lock<std::mutex> lk(hub->mu);
        auto& q = hub->box[{r.peer, rank}];
        hub->cv.wait(lk, [&] { return !q.empty(); });
        m = q.front();
        q.pop_front();
      }
      if (m->bytes != r.bytes) throw Error(NDS_ERR_OTHER, "loopback: message size mismatch");
      NDS_CUDA(cudaStreamWaitEvent(r.s, m->ready, 0));
      NDS_CUDA(cudaMemcpyAsync(r.buf, m->ptr, r.bytes, cudaMemcpyDeviceToDevice, r.s));
      NDS_CUDA(cudaEventRecord(m->done, r.s));
      {
        std::lock_guard<std::mutex> lk(hub->mu);
        m->taken = true;
      }
      hub->cv.notify_all();
    }
    recvs.clear();
    for (const Send& sd : sends) {
      {
        std::unique_lock<std::mutex> lk(hub->mu);
        hub->cv.wait(lk, [&] { return sd.m->taken; });
      }
      NDS_CUDA(cudaStreamWaitEvent(sd.s, sd.m->done, 0));
      cudaEventDestroy(sd.m->ready);  // released once the recorded work completes
      cudaEventDestroy(sd.m->done);
    }
    sends.clear();
  }
};

// dst_q[c * w_q + i] = src[c * nH + s_q + i] for all destinations q (one pass over src):
// the L_N -> L_1 pack; unpack is the inverse map. Destination q's piece starts at off[q].
struct PackMap {
  int P;
  int64_t nH, cols;
  int64_t s[64], w[64], off[64];
};

__global__ void pack_kernel(const PackMap pm, const double2* __restrict__ src, double2* __restrict__ dst, int unpack) {
  const int64_t total = pm.nH * pm.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / pm.nH, i = e % pm.nH;
    int q = 0;
    while (q + 1 < pm.P && i >= pm.s[q + 1]) ++q;
    const int64_t d = pm.off[q] + c * pm.w[q] + (i - pm.s[q]);
    if (unpack)
      dst[e] = src[d];
    else
      dst[d] = src[e];
  }
}

void pack_launch(const PackMap& pm, const double2* src, double2* dst, bool unpack, cudaStream_t s) {
  const int64_t total = pm.nH * pm.cols;
  if (total == 0) return;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 8);
  pack_kernel<<<(unsigned)blocks, 256, 0, s>>>(pm, src, dst, unpack ? 1 : 0);
  NDS_LAUNCH_CHECK();
}

void block_partition(int64_t n, int parts, std::vector<int64_t>& start, std::vector<int64_t>& size) {
  start.assign(parts, 0);
  size.assign(parts, 0);
  const int64_t base = n / parts, extra = n % parts;
  int64_t o = 0;
  for (int r = 0; r < parts; ++r) {
    size[r] = base + (r < extra ? 1 : 0);
    start[r] = o;
    o += size[r];
  }
}

// Kronecker sum of the T_j of modes [lo, hi) on their flattened (column-major) super-index.
std::vector<nds_z> kron_sum(int lo, int hi, const int64_t* dims, const nds_z* const* t, int64_t& n_out) {
  int64_t n = 1;
  for (int j = lo; j < hi; ++j) n *= dims[j];
  n_out = n;
  std::vector<nds_z> m((size_t)(n * n), nds_z{0.0, 0.0});
  for (int64_t a = 0; a < n; ++a)
    for (int64_t b = 0; b < n; ++b) {
      // nonzero only where a and b differ in at most one mode j: then T_j(a_j, b_j)
      int64_t ra = a, rb = b;
      int diff = -1, ndiff = 0;
      int64_t aj = 0, bj = 0;
      for (int j = lo; j < hi; ++j) {
        const int64_t xa = ra % dims[j], xb = rb % dims[j];
        ra /= dims[j];
        rb /= dims[j];
        if (xa != xb) {
          ++ndiff;
          diff = j;
          aj = xa;
          bj = xb;
        }
      }
      nds_z v{0.0, 0.0};
      if (ndiff == 0) {
        int64_t r = a;
        for (int j = lo; j < hi; ++j) {
          const int64_t x = r % dims[j];
          r /= dims[j];
          v.re += t[j][x + x * dims[j]].re;
          v.im += t[j][x + x * dims[j]].im;
        }
      } else if (ndiff == 1) {
        v = t[diff][aj + bj * dims[diff]];
      }
      m[(size_t)(a + b * n)] = v;
    }
  return m;
}

}  // namespace

struct nds_dist {
  nds_ctx* ctx = nullptr;
  nds_comm* comm = nullptr;
  int P = 1, rank = 0, N = 0;
  int64_t dims[NDS_MAX_MODES] = {};
  int h = 1, g = 1, gp = 1;
  int64_t nH = 1, nG = 1, nK = 1;
  std::vector<int64_t> sH, mH, sG, mG, sK, mK;
  nds::FactorSet f;  // U (four layouts) and T of the whole problem
  double tol = 0.0, min_abs_den = 0.0;
  struct Mat {
    double2* row = nullptr;
    double2* col = nullptr;
    int64_t rows = 0, cols = 0;
  };
  std::vector<Mat> head_up;                // by source rank q' (> rank, nonzero coupling)
  std::vector<std::vector<std::pair<int64_t, Mat>>> pipe_up;  // by block k: (first target block or -1 = all lower, matrix)
  std::vector<std::unique_ptr<nds_plan>> local;  // by block k: T blocks of the local solve
  std::unique_ptr<nds_plan> whole;                // one rank: the single-GPU plan path
  double2* mats = nullptr;
  double2 *ln = nullptr, *l1 = nullptr, *work = nullptr, *xbuf = nullptr, *pipe_buf[2] = {nullptr, nullptr};
  int64_t ln_size = 0, l1_size = 0, pipe_size = 0;
  cudaStream_t cs = nullptr;  // communication stream
  std::vector<cudaEvent_t> ev;
  int64_t bytes_alltoall = 0;  // per solve, this rank's all-to-all sends
  int launches = 0;

  // Does rank `lo_rank` need rank `hi_rank`'s solved blocks (T_H[lo rows, hi cols] != 0)?
  // Structural, so both sides of every transfer agree: T_1 is dense upper triangular (h = 1); a
  // binary head couples hypercube neighbours whose indices differ by one bit set in hi_rank's.
  bool couples(int lo_rank, int hi_rank) const {
    if (hi_rank <= lo_rank) return false;
    if (h == 1) return mH[lo_rank] > 0 && mH[hi_rank] > 0;
    const int64_t a = sH[lo_rank], b = sH[hi_rank];
    return __builtin_popcountll((unsigned long long)(a ^ b)) == 1 && (b & ~a) != 0;
  }

  int64_t ln_extent(int j, int r) const {  // extent of mode j in rank r's L_N slab
    if (j < N - g) return dims[j];
    return g == 1 ? mG[r] : 1;
  }
  int64_t l1_extent(int j, int q) const {
    if (j >= h) return dims[j];
    return h == 1 ? mH[q] : 1;
  }
  void ln_dims(int r, int64_t* d) const {
    for (int j = 0; j < N; ++j) d[j] = ln_extent(j, r);
  }
  void l1_dims(int q, int64_t* d) const {
    for (int j = 0; j < N; ++j) d[j] = l1_extent(j, q);
  }
};

namespace {

// Mode products of modes [lo, hi] (1-based, inclusive) on a local tensor of extents d (global
// factor set: mode j always uses U_j), src -> dst, ping-ponging through work; binary runs fused.
int apply_modes(const nds::FactorSet& f, int n_modes, const int64_t* d, int lo, int hi, bool adjoint,
                const double2* src, double2* dst, double2* work, cudaStream_t s) {
  if (lo > hi) {
    if (src != dst) {
      int64_t total = 1;
      for (int j = 0; j < n_modes; ++j) total *= d[j];
      NDS_CUDA(cudaMemcpyAsync(dst, src, (size_t)total * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    }
    return 0;
  }
  const std::vector<nds::BinGroup> groups = nds::plan_binary_groups(n_modes, d, lo - 1, hi);
  struct Pass {
    int mode, group;
  };
  std::vector<Pass> passes;
  size_t gi = 0;
  for (int j = lo; j <= hi;) {
    if (gi < groups.size() && groups[gi].first == j) {
      passes.push_back({j, (int)gi});
      j += groups[gi].count;
      ++gi;
    } else {
      passes.push_back({j, -1});
      ++j;
    }
  }
  const int np = (int)passes.size();
  const double2* cur = src;
  const bool in_place = src == dst;
  int launches = 0;
  for (int i = 0; i < np; ++i) {
    double2* out = in_place ? ((i % 2 == 0) ? work : dst) : (((np - 1 - i) % 2 == 0) ? dst : work);
    if (passes[i].group >= 0)
      nds::binary_pass_launch(f, groups[passes[i].group], adjoint, cur, out, s);
    else
      nds::mode_product_launch(f, passes[i].mode, adjoint, nds::mode_view(n_modes, d, passes[i].mode), cur, out,
                               false, s);
    ++launches;
    cur = out;
  }
  if (cur != dst) {
    int64_t total = 1;
    for (int j = 0; j < n_modes; ++j) total *= d[j];
    NDS_CUDA(cudaMemcpyAsync(dst, cur, (size_t)total * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  }
  return launches;
}

}  // namespace

namespace {

void dist_free(nds_dist* d) {
  if (!d) return;
  cudaSetDevice(d->ctx->device);
  cudaStreamSynchronize(d->ctx->stream);
  if (d->cs) cudaStreamSynchronize(d->cs);
  for (auto& p : d->local) plan_destroy_impl(p.release());
  d->local.clear();
  if (d->whole) plan_destroy_impl(d->whole.release());
  free_factors(d->f);
  for (double2* b : {d->mats, d->ln, d->l1, d->work, d->xbuf, d->pipe_buf[0]})
    if (b) cudaFree(b);
  for (auto e : d->ev) cudaEventDestroy(e);
  if (d->cs) cudaStreamDestroy(d->cs);
  delete d;
}

// Mode groups for P ranks (see the header comment). Throws when the shape does not shard.
void choose_groups(nds_dist& d) {
  const int N = d.N, P = d.P;
  if (P > 64) throw Error(NDS_ERR_INVALID, "at most 64 ranks");
  bool binary = true;
  for (int j = 0; j < N; ++j) binary = binary && d.dims[j] == 2;
  d.h = d.g = d.gp = 1;
  if (P > 1 && binary) {
    int k = 0;
    while ((1 << k) < P) ++k;
    if ((1 << k) != P) throw Error(NDS_ERR_INVALID, "all-binary problems shard over a power-of-two rank count");
    if (2 * k > N - 1) throw Error(NDS_ERR_INVALID, "too few binary modes for this rank count");
    d.h = d.g = k;
    d.gp = std::max(1, std::min(k + 1, N - k - 1));
  } else if (P > 1) {
    if (d.dims[0] < P || d.dims[N - 1] < P)
      throw Error(NDS_ERR_INVALID, "the first and last extents must be at least the number of ranks");
  }
  d.nH = d.nG = d.nK = 1;
  for (int j = 0; j < d.h; ++j) d.nH *= d.dims[j];
  for (int j = N - d.g; j < N; ++j) d.nG *= d.dims[j];
  for (int j = N - d.gp; j < N; ++j) d.nK *= d.dims[j];
  block_partition(d.nH, P, d.sH, d.mH);
  block_partition(d.nG, P, d.sG, d.mG);
  // pipeline blocks: binary -> one super-index per block; else the largest K <= 4P whose blocks
  // are whole tile edges (16 for N = 3, 8 otherwise) so the local solves keep the cubic route
  int64_t K = 1;
  if (P > 1) {
    if (binary) {
      K = d.nK;
    } else {
      const int64_t edge = N == 3 ? 16 : 8;
      for (int64_t c = std::min<int64_t>(4 * P, d.nK); c >= 2; --c)
        if (d.nK % c == 0 && (d.nK / c) % edge == 0) {
          K = c;
          break;
        }
      if (K == 1) K = std::min<int64_t>(2 * P, d.nK);  // no whole-tile blocking: pipeline anyway
    }
  }
  block_partition(d.nK, (int)K, d.sK, d.mK);
}

struct HostMat {
  std::vector<nds_z> v;  // column-major rows x cols
  int64_t rows, cols;
};

HostMat block_of(const std::vector<nds_z>& m, int64_t n, int64_t r0, int64_t rows, int64_t c0, int64_t cols,
                 bool negate, bool* nonzero) {
  HostMat h{std::vector<nds_z>((size_t)(rows * cols)), rows, cols};
  bool nz = false;
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r) {
      nds_z z = m[(size_t)((r0 + r) + (c0 + c) * n)];
      if (z.re != 0.0 || z.im != 0.0) nz = true;
      if (negate) z = nds_z{-z.re, -z.im};
      h.v[(size_t)(r + c * rows)] = z;
    }
  if (nonzero) *nonzero = nz;
  return h;
}

void dist_create_impl(nds_dist* d, const nds_z* const* u, const nds_z* const* t, double singular_tol,
                      nds_singular* sing) {
  nds_ctx* ctx = d->ctx;
  const int N = d->N;
  choose_groups(*d);
  if (d->P == 1) {  // one rank: the plan path (head / tail overlap, fused passes), no layouts
    nds_plan* p = nullptr;
    plan_create_impl(ctx, N, d->dims, u, t, singular_tol, 0u, &p, sing);
    d->whole.reset(p);
    d->tol = p->tol;
    d->min_abs_den = p->min_abs_den;
    int64_t total = 1;
    for (int j = 0; j < N; ++j) total *= d->dims[j];
    d->ln_size = d->l1_size = total;
    NDS_CUDA(cudaMalloc(&d->work, (size_t)total * sizeof(double2)));
    return;
  }
  // the whole operator's factors; one singular check of the WHOLE operator on every rank
  // (sylvester.cpp:101-103), so all ranks raise the same first offender before any exchange
  d->tol = singular_tol > 0.0 ? singular_tol : default_tol(N, d->dims, t);
  upload_factors(ctx, d->f, N, d->dims, u, t);
  int64_t bad = -1;
  nds::den_scan(d->f.geom, d->f.diag_pool, d->tol, &d->min_abs_den, &bad, ctx->stream, ctx->scratch);
  if (bad >= 0) {
    nds_singular tmp{};
    fill_singular(&tmp, N, d->dims, bad, t);
    if (sing) *sing = tmp;
    throw Error(NDS_ERR_SINGULAR, format_singular(tmp));
  }
  const int q = d->rank;
  // coupling matrices: head (Kronecker sum of the head modes) and pipe (of the pipe modes)
  int64_t nh = 0, nk = 0;
  const std::vector<nds_z> TH = kron_sum(0, d->h, d->dims, t, nh);
  const std::vector<nds_z> TK = kron_sum(N - d->gp, N, d->dims, t, nk);
  std::vector<HostMat> host_mats;
  std::vector<int> head_idx(d->P, -1);
  for (int qp = q + 1; qp < d->P; ++qp)
    if (d->couples(q, qp)) {
      head_idx[qp] = (int)host_mats.size();
      host_mats.push_back(block_of(TH, nh, d->sH[q], d->mH[q], d->sH[qp], d->mH[qp], true, nullptr));
    }
  const int K = (int)d->sK.size();
  std::vector<std::vector<std::pair<int64_t, int>>> pipe_idx(K);
  for (int k = 1; k < K; ++k) {
    std::vector<int64_t> nzb;
    for (int kk = 0; kk < k; ++kk) {
      bool nz = false;
      block_of(TK, nk, d->sK[kk], d->mK[kk], d->sK[k], d->mK[k], true, &nz);
      if (nz) nzb.push_back(kk);
    }
    if ((int)nzb.size() == k) {  // every lower block: one batched update over rows [0, sK_k)
      pipe_idx[k].push_back({-1, (int)host_mats.size()});
      host_mats.push_back(block_of(TK, nk, 0, d->sK[k], d->sK[k], d->mK[k], true, nullptr));
    } else {
      for (int64_t kk : nzb) {
        pipe_idx[k].push_back({kk, (int)host_mats.size()});
        host_mats.push_back(block_of(TK, nk, d->sK[kk], d->mK[kk], d->sK[k], d->mK[k], true, nullptr));
      }
    }
  }
  // one device pool: per matrix [row-major | column-major]
  int64_t total_m = 0;
  for (auto& hm : host_mats) total_m += 2 * hm.rows * hm.cols;
  std::vector<double2> stage((size_t)std::max<int64_t>(1, total_m));
  NDS_CUDA(cudaMalloc(&d->mats, stage.size() * sizeof(double2)));
  std::vector<nds_dist::Mat> dev;
  int64_t off = 0;
  for (auto& hm : host_mats) {
    nds_dist::Mat m;
    m.rows = hm.rows;
    m.cols = hm.cols;
    m.row = d->mats + off;
    m.col = d->mats + off + hm.rows * hm.cols;
    for (int64_t c = 0; c < hm.cols; ++c)
      for (int64_t r = 0; r < hm.rows; ++r) {
        const nds_z z = hm.v[(size_t)(r + c * hm.rows)];
        stage[(size_t)(off + r * hm.cols + c)] = make_double2(z.re, z.im);
        stage[(size_t)(off + hm.rows * hm.cols + r + c * hm.rows)] = make_double2(z.re, z.im);
      }
    off += 2 * hm.rows * hm.cols;
    dev.push_back(m);
  }
  NDS_CUDA(cudaMemcpy(d->mats, stage.data(), stage.size() * sizeof(double2), cudaMemcpyHostToDevice));
  d->head_up.assign(d->P, nds_dist::Mat{});
  for (int qp = 0; qp < d->P; ++qp)
    if (head_idx[qp] >= 0) d->head_up[qp] = dev[head_idx[qp]];
  d->pipe_up.assign(K, {});
  for (int k = 0; k < K; ++k)
    for (auto& pr : pipe_idx[k]) d->pipe_up[k].push_back({pr.first, dev[pr.second]});
  // local solves: T restricted to this rank's head block and block k's pipe block; extent-1
  // modes folded into the first remaining mode's diagonal (den is a sum over modes)
  int64_t l1d[NDS_MAX_MODES];
  d->l1_dims(q, l1d);
  for (int k = 0; k < K; ++k) {
    std::vector<int64_t> ext(N);
    std::vector<std::vector<nds_z>> tb(N);
    for (int j = 0; j < N; ++j) {
      const int64_t n = d->dims[j];
      int64_t s0 = 0, m = n;
      if (j < d->h) {
        if (d->h == 1) {
          s0 = d->sH[q];
          m = d->mH[q];
        } else {  // binary head: one super-index, this mode's bit of it
          int64_t r = d->sH[q];
          for (int i = 0; i < j; ++i) r /= d->dims[i];
          s0 = r % n;
          m = 1;
        }
      } else if (j >= N - d->gp) {
        if (d->gp == 1) {
          s0 = d->sK[k];
          m = d->mK[k];
        } else {
          int64_t r = d->sK[k];
          for (int i = N - d->gp; i < j; ++i) r /= d->dims[i];
          s0 = r % n;
          m = 1;
        }
      }
      ext[j] = m;
      tb[j].resize((size_t)(m * m));
      for (int64_t c = 0; c < m; ++c)
        for (int64_t r = 0; r < m; ++r) tb[j][(size_t)(r + c * m)] = t[j][(s0 + r) + (s0 + c) * n];
    }
    std::vector<int64_t> ld;
    std::vector<std::vector<nds_z>> lt;
    nds_z fold{0.0, 0.0};
    for (int j = 0; j < N; ++j) {
      if (ext[j] == 1) {
        fold.re += tb[j][0].re;
        fold.im += tb[j][0].im;
      } else {
        ld.push_back(ext[j]);
        lt.push_back(tb[j]);
      }
    }
    if (ld.empty()) {
      ld.push_back(1);
      lt.push_back({fold});
    } else {
      for (int64_t i = 0; i < ld[0]; ++i) {
        lt[0][(size_t)(i + i * ld[0])].re += fold.re;
        lt[0][(size_t)(i + i * ld[0])].im += fold.im;
      }
    }
    std::vector<const nds_z*> tp;
    for (auto& m : lt) tp.push_back(m.data());
    std::unique_ptr<nds_plan> p(new nds_plan);
    p->ctx = ctx;
    p->n_modes = (int)ld.size();
    std::memcpy(p->dims, ld.data(), ld.size() * sizeof(int64_t));
    p->total = 1;
    for (int64_t e : ld) p->total *= e;
    p->tol = d->tol;
    upload_factors(ctx, p->f, p->n_modes, p->dims, nullptr, tp.data());
    build_solver(p.get());
    d->local.push_back(std::move(p));
  }
  // buffers
  int64_t lnd[NDS_MAX_MODES];
  d->ln_dims(q, lnd);
  d->ln_size = d->l1_size = 1;
  for (int j = 0; j < N; ++j) {
    d->ln_size *= lnd[j];
    d->l1_size *= l1d[j];
  }
  int64_t Mp = 1;  // modes strictly between the head and the pipe groups
  for (int j = d->h; j < N - d->gp; ++j) Mp *= d->dims[j];
  int64_t maxk = 0, src_rows = 0;
  for (int64_t m : d->mK) maxk = std::max(maxk, m);
  for (int qp = q + 1; qp < d->P; ++qp)
    if (d->head_up[qp].row) src_rows += d->mH[qp];
  d->pipe_size = std::max<int64_t>(1, src_rows * Mp * maxk);
  const int64_t big = std::max(d->ln_size, d->l1_size);
  NDS_CUDA(cudaMalloc(&d->ln, (size_t)big * sizeof(double2)));
  NDS_CUDA(cudaMalloc(&d->l1, (size_t)big * sizeof(double2)));
  NDS_CUDA(cudaMalloc(&d->work, (size_t)big * sizeof(double2)));
  NDS_CUDA(cudaMalloc(&d->xbuf, (size_t)big * sizeof(double2)));
  NDS_CUDA(cudaMalloc(&d->pipe_buf[0], (size_t)(2 * d->pipe_size) * sizeof(double2)));
  d->pipe_buf[1] = d->pipe_buf[0] + d->pipe_size;
  int lo = 0, hi = 0;
  NDS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  NDS_CUDA(cudaStreamCreateWithPriority(&d->cs, cudaStreamNonBlocking, hi));
  d->ev.resize(2 * K + 8);
  for (auto& e : d->ev) NDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // traffic per solve (this rank's sends): both all-to-alls and the pipeline forwarding
  int64_t Mg = 1;  // modes strictly between the head and the tail groups
  for (int j = d->h; j < N - d->g; ++j) Mg *= d->dims[j];
  for (int r = 0; r < d->P; ++r)
    if (r != q) d->bytes_alltoall += 16 * (d->mH[r] * Mg * d->mG[q] + d->mH[q] * Mg * d->mG[r]);
}

int dist_solve_impl(nds_dist* d, const double2* b, double2* x) {
  nds_ctx* ctx = d->ctx;
  if (d->whole) {
    d->launches = execute(d->whole.get(), b, x, d->work, nullptr);
    return d->launches;
  }
  const int N = d->N, q = d->rank, P = d->P;
  const int K = (int)d->sK.size();
  cudaStream_t s = ctx->stream, cs = d->cs;
  nds_comm* comm = d->comm;
  int launches = 0;
  int64_t lnd[NDS_MAX_MODES], l1d[NDS_MAX_MODES];
  d->ln_dims(q, lnd);
  d->l1_dims(q, l1d);
  int64_t Mg = 1, Mp = 1;
  for (int j = d->h; j < N - d->g; ++j) Mg *= d->dims[j];
  for (int j = d->h; j < N - d->gp; ++j) Mp *= d->dims[j];
  cudaEvent_t* E = d->ev.data() + 2 * K;
  auto cs_wait = [&](cudaEvent_t e, cudaStream_t from, cudaStream_t to) {
    NDS_CUDA(cudaEventRecord(e, from));
    NDS_CUDA(cudaStreamWaitEvent(to, e, 0));
  };
  // pieces of the L_N <-> L_1 exchange: to / from rank r, (head block of the L_1 owner) x Mg x
  // (tail block of the L_N owner)
  std::vector<int64_t> ln_piece_off(P), ln_piece_len(P);
  {
    int64_t o = 0;
    for (int r = 0; r < P; ++r) {
      ln_piece_off[r] = o;
      ln_piece_len[r] = d->mH[r] * Mg * d->mG[q];
      o += ln_piece_len[r];
    }
  }
  PackMap pm{};
  pm.P = P;
  pm.nH = d->nH;
  pm.cols = Mg * d->mG[q];
  for (int r = 0; r < P; ++r) {
    pm.s[r] = d->sH[r];
    pm.w[r] = d->mH[r];
    pm.off[r] = ln_piece_off[r];
  }
  // 1. forward modes outside the tail group, local in L_N
  launches += apply_modes(d->f, N, lnd, 1, N - d->g, true, b, d->ln, d->work, s);
  // 2. L_N -> L_1
  if (P > 1) {
    pack_launch(pm, d->ln, d->xbuf, false, s);
    ++launches;
    cs_wait(E[0], s, cs);
    comm->group_begin();
    for (int r = 0; r < P; ++r) {
      if (r == q) continue;
      if (ln_piece_len[r] > 0) comm->send(d->xbuf + ln_piece_off[r], (size_t)ln_piece_len[r] * 16, r, cs);
      const int64_t n_in = d->mH[q] * Mg * d->mG[r];
      if (n_in > 0) comm->recv(d->l1 + d->sG[r] * d->mH[q] * Mg, (size_t)n_in * 16, r, cs);
    }
    comm->group_end();
    if (ln_piece_len[q] > 0)
      NDS_CUDA(cudaMemcpyAsync(d->l1 + d->sG[q] * d->mH[q] * Mg, d->xbuf + ln_piece_off[q],
                               (size_t)ln_piece_len[q] * 16, cudaMemcpyDeviceToDevice, s));
    cs_wait(E[1], cs, s);
  } else {
    NDS_CUDA(cudaMemcpyAsync(d->l1, d->ln, (size_t)d->l1_size * 16, cudaMemcpyDeviceToDevice, s));
  }
  // 3. forward modes of the tail group, local in L_1
  launches += apply_modes(d->f, N, l1d, N - d->g + 1, N, true, d->l1, d->l1, d->work, s);
  // 4. pipelined triangular solve in place on l1
  const int64_t plane = d->mH[q] * Mp;  // entries per pipe super-index
  std::vector<int> higher, lower;
  for (int qp = P - 1; qp > q; --qp)
    if (d->head_up[qp].row) higher.push_back(qp);
  for (int qq = q - 1; qq >= 0; --qq)
    if (d->couples(qq, q)) lower.push_back(qq);
  auto recv_block = [&](int k) {
    if (higher.empty()) return;
    double2* buf = d->pipe_buf[k & 1];
    int64_t o = 0;
    comm->group_begin();
    for (int qp : higher) {
      const int64_t n_in = d->mH[qp] * Mp * d->mK[k];
      comm->recv(buf + o, (size_t)n_in * 16, qp, cs);
      o += n_in;
    }
    comm->group_end();
  };
  cs_wait(E[2], s, cs);
  if (P > 1) recv_block(K - 1);
  NDS_CUDA(cudaEventRecord(d->ev[K - 1], cs));  // R[K-1]
  for (int k = K - 1; k >= 0; --k) {
    double2* blk = d->l1 + d->sK[k] * plane;
    NDS_CUDA(cudaStreamWaitEvent(s, d->ev[k], 0));  // R[k]
    // head couplings from the higher ranks' block k (descending rank: fixed order)
    {
      int64_t o = 0;
      for (int qp : higher) {
        const nds_dist::Mat& m = d->head_up[qp];
        const nds::ModeView v{1, d->mH[qp], Mp * d->mK[k]};
        nds::mode_product_matrix_launch(m.row, m.col, v, d->pipe_buf[k & 1] + o, blk, true, s, d->mH[q]);
        ++launches;
        o += d->mH[qp] * Mp * d->mK[k];
      }
    }
    launches += launch_solver(d->local[k].get(), blk, s, nullptr);
    NDS_CUDA(cudaEventRecord(d->ev[K + k], s));  // S[k]
    if (P > 1 && (!lower.empty() || (k > 0 && !higher.empty()))) {
      NDS_CUDA(cudaStreamWaitEvent(cs, d->ev[K + k], 0));
      comm->group_begin();
      for (int qq : lower) comm->send(blk, (size_t)(plane * d->mK[k]) * 16, qq, cs);
      if (k > 0) recv_block(k - 1);
      comm->group_end();
    }
    if (k > 0) NDS_CUDA(cudaEventRecord(d->ev[k - 1], cs));  // R[k-1]
    // pipe couplings of block k into the lower blocks of this rank
    for (auto& pr : d->pipe_up[k]) {
      const nds_dist::Mat& m = pr.second;
      const nds::ModeView v{plane, d->mK[k], 1};
      double2* dst = pr.first < 0 ? d->l1 : d->l1 + d->sK[pr.first] * plane;
      nds::mode_product_matrix_launch(m.row, m.col, v, blk, dst, true, s, m.rows);
      ++launches;
    }
  }
  cs_wait(E[3], cs, s);  // the last sends have read Y before the inverse overwrites it
  // 5. inverse modes outside the head group, local in L_1
  launches += apply_modes(d->f, N, l1d, d->h + 1, N, false, d->l1, d->l1, d->work, s);
  // 6. L_1 -> L_N
  if (P > 1) {
    cs_wait(E[4], s, cs);
    comm->group_begin();
    for (int r = 0; r < P; ++r) {
      if (r == q) continue;
      const int64_t n_out = d->mH[q] * Mg * d->mG[r];
      if (n_out > 0) comm->send(d->l1 + d->sG[r] * d->mH[q] * Mg, (size_t)n_out * 16, r, cs);
      if (ln_piece_len[r] > 0) comm->recv(d->xbuf + ln_piece_off[r], (size_t)ln_piece_len[r] * 16, r, cs);
    }
    comm->group_end();
    if (ln_piece_len[q] > 0)
      NDS_CUDA(cudaMemcpyAsync(d->xbuf + ln_piece_off[q], d->l1 + d->sG[q] * d->mH[q] * Mg,
                               (size_t)ln_piece_len[q] * 16, cudaMemcpyDeviceToDevice, s));
    cs_wait(E[5], cs, s);
    pack_launch(pm, d->xbuf, d->ln, true, s);
    ++launches;
  } else {
    NDS_CUDA(cudaMemcpyAsync(d->ln, d->l1, (size_t)d->ln_size * 16, cudaMemcpyDeviceToDevice, s));
  }
  // 7. inverse modes of the head group, local in L_N
  launches += apply_modes(d->f, N, lnd, 1, d->h, false, d->ln, x, d->work, s);
  d->launches = launches;
  return launches;
}

}  // namespace

extern "C" {

int nds_comm_unique_id(void* id_out) {
  return guarded(nullptr, [&] {
    if (!id_out) throw Error(NDS_ERR_INVALID, "null id buffer");
    ncclUniqueId id;
    nccl_check(nccl_api().get_unique_id(&id), "get unique id");
    static_assert(sizeof(ncclUniqueId) == NDS_COMM_ID_BYTES, "NCCL unique id size");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int nds_comm_create_nccl(nds_comm** out, int device, int rank, int world, const void* id) {
  return guarded(nullptr, [&] {
    if (!out || !id || world < 1 || rank < 0 || rank >= world) throw Error(NDS_ERR_INVALID, "bad communicator arguments");
    *out = nullptr;
    NDS_CUDA(cudaSetDevice(device));
    std::unique_ptr<NcclComm> c(new NcclComm);
    c->rank = rank;
    c->world = world;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl_api().comm_init_rank(&c->comm, world, uid, rank), "comm init");
    *out = c.release();
  });
}

int nds_comm_create_loopback(int world, nds_comm** out) {
  return guarded(nullptr, [&] {
    if (!out || world < 1) throw Error(NDS_ERR_INVALID, "bad loopback arguments");
    auto hub = std::make_shared<LoopHub>();
    for (int r = 0; r < world; ++r) {
      auto* c = new LoopComm;
      c->rank = r;
      c->world = world;
      c->hub = hub;
      out[r] = c;
    }
  });
}

void nds_comm_destroy(nds_comm* c) { delete c; }

int nds_dist_create(nds_ctx* ctx, nds_comm* comm, int n_modes, const int64_t* dims, const nds_z* const* u,
                    const nds_z* const* t, double singular_tol, nds_dist** out, nds_singular* sing) {
  if (!ctx) return NDS_ERR_INVALID;
  return guarded(ctx, [&] {
    if (!out) throw Error(NDS_ERR_INVALID, "out is null");
    *out = nullptr;
    checked_total(n_modes, dims, 2);
    require_ptrs(n_modes, u, "u");
    require_ptrs(n_modes, t, "t");
    ensure_device(ctx);
    std::unique_ptr<nds_dist, void (*)(nds_dist*)> d(new nds_dist, dist_free);
    d->ctx = ctx;
    d->comm = comm;
    d->P = comm ? comm->world : 1;
    d->rank = comm ? comm->rank : 0;
    d->N = n_modes;
    std::memcpy(d->dims, dims, n_modes * sizeof(int64_t));
    dist_create_impl(d.get(), u, t, singular_tol, sing);
    NDS_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = d.release();
  });
}

void nds_dist_destroy(nds_dist* d) { dist_free(d); }

int nds_dist_slab(const nds_dist* d, int rank, int64_t* offset, int64_t* count) {
  if (!d || rank < 0 || rank >= d->P) return NDS_ERR_INVALID;
  int64_t head = 1;
  for (int j = 0; j < d->N - d->g; ++j) head *= d->dims[j];
  if (offset) *offset = d->sG[rank] * head;
  if (count) *count = d->mG[rank] * head;
  return NDS_OK;
}

int nds_dist_info(const nds_dist* d, nds_dist_info_t* info) {
  if (!d || !info) return NDS_ERR_INVALID;
  std::memset(info, 0, sizeof(*info));
  info->ranks = d->P;
  info->rank = d->rank;
  info->head_modes = d->h;
  info->tail_modes = d->g;
  info->pipe_modes = d->gp;
  info->pipe_blocks = (int)d->sK.size();
  info->local_solve_path = -1;
  if (!d->local.empty()) info->local_solve_path = nds_plan_solve_path(d->local[0].get());
  if (d->whole) info->local_solve_path = nds_plan_solve_path(d->whole.get());
  info->alltoall_bytes = d->bytes_alltoall;
  int64_t Mp = 1;
  for (int j = d->h; j < d->N - d->gp; ++j) Mp *= d->dims[j];
  int lower = 0;
  for (int qq = 0; qq < d->rank; ++qq) lower += d->couples(qq, d->rank) ? 1 : 0;
  info->pipeline_bytes = 16 * d->mH[d->rank] * Mp * d->nK * lower;
  info->launches = d->launches;
  info->min_abs_denominator = d->min_abs_den;
  return NDS_OK;
}

int nds_dist_solve(nds_dist* d, const nds_z* d_b, nds_z* d_x) {
  if (!d) return NDS_ERR_INVALID;
  return guarded(d->ctx, [&] {
    if (!d_b || !d_x) throw Error(NDS_ERR_INVALID, "null device tensor pointer");
    ensure_device(d->ctx);
    dist_solve_impl(d, (const double2*)d_b, (double2*)d_x);
  });
}

// One process, n devices: one host thread, context and NCCL communicator per device; B and X
// host tensors (column-major); each device takes its L_N slab (a contiguous range of B).
int nds_solve_multi(int n_devices, const int* devices, int n_modes, const int64_t* dims, const nds_z* const* u,
                    const nds_z* const* t, const nds_z* b, nds_z* x, double singular_tol, nds_singular* sing) {
  return guarded(nullptr, [&] {
    if (n_devices < 1 || !devices || !b || !x) throw Error(NDS_ERR_INVALID, "bad multi-device arguments");
    checked_total(n_modes, dims, 2);
    require_ptrs(n_modes, u, "u");
    require_ptrs(n_modes, t, "t");
    ncclUniqueId id{};
    if (n_devices > 1) nccl_check(nccl_api().get_unique_id(&id), "get unique id");
    std::vector<int> rc(n_devices, NDS_OK);
    std::vector<std::string> err(n_devices);
    std::vector<nds_singular> sg(n_devices);
    auto worker = [&](int r) {
      nds_ctx* ctx = nullptr;
      nds_comm* comm = nullptr;
      nds_dist* d = nullptr;
      double2 *db = nullptr, *dx = nullptr;
      auto fail = [&](int code, const std::string& m) {
        rc[r] = code;
        err[r] = m;
      };
      int c = nds_ctx_create(&ctx, devices[r]);
      if (c) return fail(c, nds_last_error(nullptr));
      if (n_devices > 1) c = nds_comm_create_nccl(&comm, devices[r], r, n_devices, &id);
      if (!c) c = nds_dist_create(ctx, comm, n_modes, dims, u, t, singular_tol, &d, &sg[r]);
      if (!c) {
        int64_t off = 0, cnt = 0;
        nds_dist_slab(d, r, &off, &cnt);
        if (cudaMalloc(&db, (size_t)std::max<int64_t>(1, cnt) * 16) != cudaSuccess ||
            cudaMalloc(&dx, (size_t)std::max<int64_t>(1, cnt) * 16) != cudaSuccess) {
          c = NDS_ERR_NOMEM;
        } else {
          cudaMemcpyAsync(db, b + off, (size_t)cnt * 16, cudaMemcpyHostToDevice, ctx->stream);
          c = nds_dist_solve(d, (const nds_z*)db, (nds_z*)dx);
          if (!c) {
            cudaMemcpyAsync(x + off, dx, (size_t)cnt * 16, cudaMemcpyDeviceToHost, ctx->stream);
            if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) c = NDS_ERR_CUDA;
          }
        }
      }
      if (c) fail(c, ctx ? nds_last_error(ctx) : nds_last_error(nullptr));
      if (db) cudaFree(db);
      if (dx) cudaFree(dx);
      nds_dist_destroy(d);
      nds_comm_destroy(comm);
      nds_ctx_destroy(ctx);
    };
    std::vector<std::thread> th;
    for (int r = 1; r < n_devices; ++r) th.emplace_back(worker, r);
    worker(0);
    for (auto& tt : th) tt.join();
    for (int r = 0; r < n_devices; ++r)
      if (rc[r]) {
        if (rc[r] == NDS_ERR_SINGULAR && sing) *sing = sg[r];
        throw Error(rc[r], "device " + std::to_string(devices[r]) + ": " + err[r]);
      }
  });
}

}  // extern "C"
