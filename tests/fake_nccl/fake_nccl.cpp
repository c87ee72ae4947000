// fake_nccl.cpp — TEST INFRASTRUCTURE, never linked into the product.
//
// A host-staged stand-in for the handful of NCCL entry points
// libraybos_gpu.so dlopens (capi.cpp NcclApi), so the library's multi-GPU code
// paths — rb_create(n > 1) / rb_create_devices, rb_create_rank, the grouped
// reduce and all-reduces of rb_trace / rb_trace_bos_pair — can execute on a
// box with ONE GPU.  Selected with RAYBOS_NCCL_LIB=<path to this .so>.
//
// Why not real NCCL on one GPU: NCCL refuses two ranks on the same device, and
// even if it did not, collective kernels of several ranks on one GPU wait on
// each other (the pool's profiling guide forbids that).  This stand-in never
// launches a kernel: every collective synchronises the caller's stream, copies
// the buffers to the host, sums them in rank order and copies the result back.
//
//  * ncclCommInitAll (in-process): the communicators form a clique; the
//    collectives of one ncclGroupStart/End are matched per clique in call
//    order and executed at ncclGroupEnd.  Duplicate device ordinals are allowed.
//  * ncclGetUniqueId / ncclCommInitRank (one process per rank): the id carries
//    a rendezvous directory; each collective writes this rank's bytes to a file
//    there, and the ranks that need the result poll for the other ranks' files
//    (host-side waits only).
#include <cuda_runtime.h>
#include <nccl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

struct Clique {
  std::vector<ncclComm*> members;  // by rank
};

struct ncclComm {
  int nranks = 1, rank = 0, device = 0;
  std::shared_ptr<Clique> clique;  // in-process
  std::string dir;                 // multi-process rendezvous
  uint64_t seq = 0;
};

namespace {

struct Op {
  bool all;
  const void* send;
  void* recv;
  size_t count;
  ncclDataType_t dt;
  ncclRedOp_t op;
  int root;
  ncclComm_t comm;
  cudaStream_t stream;
};

thread_local int g_depth = 0;
thread_local std::vector<Op> g_pending;

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

template <typename T>
void combine_t(void* acc, const void* x, size_t n, ncclRedOp_t op) {
  T* a = static_cast<T*>(acc);
  const T* b = static_cast<const T*>(x);
  for (size_t i = 0; i < n; ++i) a[i] = op == ncclMax ? (b[i] > a[i] ? b[i] : a[i]) : a[i] + b[i];
}

bool combine(void* acc, const void* x, size_t n, ncclDataType_t t, ncclRedOp_t op) {
  if (op != ncclSum && op != ncclMax) return false;
  switch (t) {
    case ncclInt32: combine_t<int32_t>(acc, x, n, op); return true;
    case ncclUint32: combine_t<uint32_t>(acc, x, n, op); return true;
    case ncclInt64: combine_t<int64_t>(acc, x, n, op); return true;
    case ncclUint64: combine_t<uint64_t>(acc, x, n, op); return true;
    case ncclFloat64: combine_t<double>(acc, x, n, op); return true;
    case ncclFloat32: combine_t<float>(acc, x, n, op); return true;
    default: return false;
  }
}

bool to_host(const Op& o, std::vector<char>& h) {
  h.resize(o.count * type_size(o.dt));
  if (cudaSetDevice(o.comm->device) != cudaSuccess) return false;
  if (cudaStreamSynchronize(o.stream) != cudaSuccess) return false;
  return h.empty() || cudaMemcpy(h.data(), o.send, h.size(), cudaMemcpyDeviceToHost) == cudaSuccess;
}

bool to_device(const Op& o, const std::vector<char>& h) {
  if (cudaSetDevice(o.comm->device) != cudaSuccess) return false;
  return h.empty() || cudaMemcpy(o.recv, h.data(), h.size(), cudaMemcpyHostToDevice) == cudaSuccess;
}

// One matched collective across a clique (ops[r] is rank r's call).
ncclResult_t run_clique(const std::vector<const Op*>& ops) {
  std::vector<std::vector<char>> h(ops.size());
  for (size_t r = 0; r < ops.size(); ++r)
    if (!to_host(*ops[r], h[r])) return ncclUnhandledCudaError;
  std::vector<char> acc = h[0];
  for (size_t r = 1; r < ops.size(); ++r)
    if (!combine(acc.data(), h[r].data(), ops[0]->count, ops[0]->dt, ops[0]->op))
      return ncclInvalidArgument;
  for (size_t r = 0; r < ops.size(); ++r)
    if (ops[r]->all || static_cast<int>(r) == ops[r]->root)
      if (!to_device(*ops[r], acc)) return ncclUnhandledCudaError;
  return ncclSuccess;
}

std::string slot(const ncclComm* c, uint64_t seq, int rank) {
  return c->dir + "/s" + std::to_string(seq) + "_r" + std::to_string(rank);
}

ncclResult_t run_dist(const Op& o) {
  ncclComm* c = o.comm;
  std::vector<char> mine;
  if (!to_host(o, mine)) return ncclUnhandledCudaError;
  const uint64_t seq = c->seq++;
  {
    const std::string tmp = slot(c, seq, c->rank) + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return ncclSystemError;
    const bool ok = mine.empty() || std::fwrite(mine.data(), 1, mine.size(), f) == mine.size();
    std::fclose(f);
    if (!ok || std::rename(tmp.c_str(), slot(c, seq, c->rank).c_str()) != 0) return ncclSystemError;
  }
  if (!o.all && c->rank != o.root) return ncclSuccess;
  std::vector<char> acc;
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(300);
  for (int r = 0; r < c->nranks; ++r) {
    std::vector<char> x;
    if (r == c->rank) {
      x = mine;
    } else {
      const std::string p = slot(c, seq, r);
      for (;;) {
        FILE* f = std::fopen(p.c_str(), "rb");
        if (f) {
          x.resize(mine.size());
          const size_t got = x.empty() ? 0 : std::fread(x.data(), 1, x.size(), f);
          std::fclose(f);
          if (got != x.size()) return ncclSystemError;
          break;
        }
        if (std::chrono::steady_clock::now() > deadline) return ncclSystemError;
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
    }
    if (r == 0) acc = x;
    else if (!combine(acc.data(), x.data(), o.count, o.dt, o.op)) return ncclInvalidArgument;
  }
  return to_device(o, acc) ? ncclSuccess : ncclUnhandledCudaError;
}

ncclResult_t execute(std::vector<Op>& ops) {
  // in-process: per clique, the k-th call of every member forms one collective
  std::map<Clique*, std::vector<std::vector<const Op*>>> per;  // clique -> rank -> ops
  for (const Op& o : ops) {
    if (o.comm->clique) {
      auto& v = per[o.comm->clique.get()];
      v.resize(o.comm->clique->members.size());
      v[o.comm->rank].push_back(&o);
    } else {
      if (ncclResult_t r = run_dist(o)) return r;
    }
  }
  for (auto& kv : per) {
    auto& ranks = kv.second;
    const size_t k = ranks[0].size();
    for (auto& r : ranks)
      if (r.size() != k) return ncclInvalidUsage;  // a member skipped a collective
    for (size_t j = 0; j < k; ++j) {
      std::vector<const Op*> set;
      for (auto& r : ranks) set.push_back(r[j]);
      if (ncclResult_t r = run_clique(set)) return r;
    }
  }
  return ncclSuccess;
}

ncclResult_t submit(const Op& o) {
  if (g_depth > 0) {
    g_pending.push_back(o);
    return ncclSuccess;
  }
  std::vector<Op> one{o};
  return execute(one);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetVersion(int* version) {
  if (version) *version = 0;  // 0 marks the stand-in
  return ncclSuccess;
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  const char* base = std::getenv("RAYBOS_FAKE_NCCL_DIR");
  std::string tmpl = std::string(base && *base ? base : "/tmp") + "/fake_nccl_XXXXXX";
  std::vector<char> buf(tmpl.begin(), tmpl.end());
  buf.push_back('\0');
  if (!mkdtemp(buf.data())) return ncclSystemError;
  if (std::strlen(buf.data()) >= sizeof(id->internal)) return ncclInternalError;
  std::memset(id->internal, 0, sizeof(id->internal));
  std::strcpy(id->internal, buf.data());
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  auto* c = new ncclComm();
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  c->dir.assign(id.internal, strnlen(id.internal, sizeof(id.internal)));
  struct stat st;
  if (stat(c->dir.c_str(), &st) != 0) {
    delete c;
    return ncclInvalidArgument;
  }
  *comm = c;
  return ncclSuccess;
}

ncclResult_t ncclCommInitAll(ncclComm_t* comms, int ndev, const int* devlist) {
  if (!comms || ndev < 1) return ncclInvalidArgument;
  auto cl = std::make_shared<Clique>();
  for (int i = 0; i < ndev; ++i) {
    auto* c = new ncclComm();
    c->nranks = ndev;
    c->rank = i;
    c->device = devlist ? devlist[i] : i;
    c->clique = cl;
    cl->members.push_back(c);
    comms[i] = c;
  }
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete comm;
  return ncclSuccess;
}

ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) {
  if (!comm || !count) return ncclInvalidArgument;
  *count = comm->nranks;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++g_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (g_depth == 0) return ncclInvalidUsage;
  if (--g_depth > 0) return ncclSuccess;
  std::vector<Op> ops;
  ops.swap(g_pending);
  return execute(ops);
}

ncclResult_t ncclReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                        ncclRedOp_t op, int root, ncclComm_t comm, cudaStream_t stream) {
  if (!comm) return ncclInvalidArgument;
  return submit(Op{false, sendbuff, recvbuff, count, datatype, op, root, comm, stream});
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count,
                           ncclDataType_t datatype, ncclRedOp_t op, ncclComm_t comm,
                           cudaStream_t stream) {
  if (!comm) return ncclInvalidArgument;
  return submit(Op{true, sendbuff, recvbuff, count, datatype, op, 0, comm, stream});
}

}  // extern "C"
