// The dim-sharded memory group behind the C ABI (§3.1.2, P:159-167,
// Fig. 2): "The memory values are sharded across the embedding
// dimension.  At each step, the indices are gathered from the process group,
// each worker does a lookup and then aggregates the portion of embeddings in
// its own shard.  After this, each worker gathers the partial embeddings
// corresponding to its own portion of the indices."
//
// A group owns its transport: NCCL (ml_group_init; one process per GPU, the
// 128-byte unique id broadcast by the caller), an in-process hub whose G
// ranks are host threads on one device (ml_group_init_hub; the collectives
// are host-synchronised copies, so no kernel ever waits on another -- the
// single-GPU test harness of exactly this protocol code), or a loopback (one
// rank with the network removed: t_ref(G) of SURVEY §8(e) through this code
// path, ml_group_init_loopback).
//
// Forward (mode P, the paper's): (idx, w) packed into one all-gather; own
// positions sorted for the backward's inverse map on a preparation stream
// (the sorted lists all-gathered and merged later: the map is built once per
// group); the bag forward over all group tokens on this rank's [N, dv/G]
// slice as one launch, its G token blocks sent to their owners by one
// all-to-all, and the owner interleaves the G slices (+ the silu gate).  Mode
// N (north-star wording): the blocks are all-gathered instead and every rank
// holds every token's full row.  With peer memory (ml_group_set_p2p) the bag
// kernel stores every block straight into its owner's exchange region.
// Backward (reading Q14): the dy slices travel back by one all-to-all (or are
// stored into the owners' regions), the sorted segmented reduction runs on
// the local slice (dV never leaves the rank), and the partial dw (a dot over
// dv/G columns) is reduce-scattered to the token owners (or summed by them
// from their regions in rank order).
#include "internal.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#define ML_API_BEGIN_X try {
#define ML_API_END_X                                                            \
  }                                                                             \
  catch (const std::exception& e) {                                             \
    return ::ml::fail(ML_ERR_CUDA, std::string("internal exception: ") + e.what()); \
  }                                                                             \
  catch (...) {                                                                 \
    return ::ml::fail(ML_ERR_CUDA, "internal exception");                       \
  }

namespace ml {
namespace {

// ------------------------------------------------------------ NCCL (dlopen)
// NCCL is resolved at run time (the process's libnccl.so.2 -- torch's, when
// torch.distributed loaded it), so the library loads without it and only
// the NCCL group calls fail (ML_ERR_NCCL) when it is absent.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [h](const char* n) { return dlsym(h, n); };
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(sym("ncclAllGather"));
    api.reduceScatter = reinterpret_cast<decltype(api.reduceScatter)>(sym("ncclReduceScatter"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allGather &&
             api.reduceScatter && api.send && api.recv && api.groupStart && api.groupEnd &&
             api.errorString;
  });
  return api;
}

#define ML_NCCL_TRY(expr)                                                              \
  do {                                                                                 \
    ncclResult_t _r = (expr);                                                          \
    if (_r != ncclSuccess)                                                             \
      return ::ml::fail(ML_ERR_NCCL, std::string(#expr) + ": " + nccl().errorString(_r)); \
  } while (0)

// ------------------------------------------------------------ transports
struct Transport {
  int G = 1, rank = 0;
  virtual ~Transport() {}
  // recv [G][bytes] <- every rank's send [bytes]
  virtual mlStatus all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // recv[g] <- rank g's send[rank] (send, recv: [G][bytes])
  virtual mlStatus all_to_all(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // recv [count] = sum over ranks of their send[rank] (send: [G][count] fp32)
  virtual mlStatus reduce_scatter_f32(const float* send, float* recv, size_t count,
                                      cudaStream_t s) = 0;
  // one ring step: send -> rank `to`, recv <- rank `from` (bytes each)
  virtual bool has_p2p() const { return false; }
  virtual mlStatus sendrecv(const void*, int, void*, int, size_t, cudaStream_t) {
    return fail(ML_ERR_UNSUPPORTED, "transport: no point-to-point steps");
  }
  // Peer memory (the fused exchange): every rank owns an exchange region that
  // the other ranks' kernels store into directly.  peer_setup is collective
  // (all ranks, same bytes); peer_region(g) = rank g's region as addressed by
  // this rank; peer_barrier: every peer-memory store issued on s so far is
  // visible to its target, and every peer's stores to this rank are visible
  // to the work that follows on s.
  virtual bool has_peer_mem() const { return false; }
  virtual mlStatus peer_setup(size_t, cudaStream_t) {
    return fail(ML_ERR_UNSUPPORTED, "transport: no peer memory");
  }
  virtual char* peer_region(int) { return nullptr; }
  virtual mlStatus peer_barrier(cudaStream_t) {
    return fail(ML_ERR_UNSUPPORTED, "transport: no peer memory");
  }
};

constexpr size_t kPeerFlagBytes = 4096;    // head of every exchange region: G epoch flags

// one warp: release this rank's stores (epoch flag written into every peer's
// region), then acquire every peer's (wait for their flags); bounded spin
__global__ void p2p_barrier_kernel(uint64_t* const* peer_flags, uint64_t* my_flags, int G, int rank,
                                   uint64_t epoch) {
  const int g = threadIdx.x;
  const bool peer = g < G && g != rank;
  if (peer) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flags[g] + rank), "l"(epoch)
                 : "memory");
  }
  __syncwarp();
  if (peer) {
    uint64_t v = 0;
    for (uint32_t spins = 0;; ++spins) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + g) : "memory");
      if (v >= epoch) break;
      if (spins > (1u << 26)) __trap();     // ~7 s: a peer never arrived
      __nanosleep(100);
    }
  }
  __syncwarp();
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  // peer memory: a cudaMalloc'd region per rank, mapped into the other ranks
  // with CUDA IPC (NVLink / NVSwitch peer access); epoch flags at its head
  bool peer_on = false;
  char* region = nullptr;
  size_t region_bytes = 0;
  std::vector<char*> peers;
  uint64_t** d_peer_flags = nullptr;
  uint64_t epoch = 0;
  uint8_t* d_sync = nullptr;      // [G] bytes: a 1-byte all-gather as a barrier
  ~NcclTransport() override {
    release_peers();
    if (d_sync) cudaFree(d_sync);
    if (comm) nccl().commDestroy(comm);
  }
  mlStatus nccl_barrier(cudaStream_t s) {
    if (!d_sync) ML_CUDA_TRY(cudaMalloc(&d_sync, size_t(G)));
    ML_NCCL_TRY(nccl().allGather(d_sync + rank, d_sync, 1, ncclUint8, comm, s));
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    return ML_OK;
  }
  void release_peers() {
    for (int g = 0; g < int(peers.size()); ++g)
      if (g != rank && peers[size_t(g)]) cudaIpcCloseMemHandle(peers[size_t(g)]);
    peers.clear();
    if (region) cudaFree(region);
    if (d_peer_flags) cudaFree(d_peer_flags);
    region = nullptr;
    d_peer_flags = nullptr;
    region_bytes = 0;
  }
  bool has_peer_mem() const override { return peer_on && G > 1; }
  char* peer_region(int g) override { return peers[size_t(g)]; }
  mlStatus peer_setup(size_t bytes, cudaStream_t s) override {
    if (bytes <= region_bytes) return ML_OK;      // every rank decides alike (same shapes)
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    // nobody may still write into the old regions: a collective as a barrier
    if (region) {
      ML_CUDA_TRY(cudaDeviceSynchronize());
      ML_TRY(nccl_barrier(s));
    }
    release_peers();
    ML_CUDA_TRY(cudaMalloc(&region, bytes));
    ML_CUDA_TRY(cudaMemset(region, 0, kPeerFlagBytes));
    region_bytes = bytes;
    cudaIpcMemHandle_t mine;
    ML_CUDA_TRY(cudaIpcGetMemHandle(&mine, region));
    char* d_handles = nullptr;
    ML_CUDA_TRY(cudaMalloc(&d_handles, sizeof(cudaIpcMemHandle_t) * size_t(G)));
    ML_CUDA_TRY(cudaMemcpyAsync(d_handles + sizeof(mine) * size_t(rank), &mine, sizeof(mine),
                                cudaMemcpyHostToDevice, s));
    ML_NCCL_TRY(nccl().allGather(d_handles + sizeof(mine) * size_t(rank), d_handles, sizeof(mine),
                                 ncclUint8, comm, s));
    std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(G));
    ML_CUDA_TRY(cudaMemcpyAsync(all.data(), d_handles, sizeof(mine) * size_t(G), cudaMemcpyDeviceToHost, s));
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(d_handles);
    peers.assign(size_t(G), nullptr);
    std::vector<uint64_t*> flags(static_cast<size_t>(G));
    for (int g = 0; g < G; ++g) {
      if (g == rank) {
        peers[size_t(g)] = region;
      } else {
        void* p = nullptr;
        ML_CUDA_TRY(cudaIpcOpenMemHandle(&p, all[size_t(g)], cudaIpcMemLazyEnablePeerAccess));
        peers[size_t(g)] = static_cast<char*>(p);
      }
      flags[size_t(g)] = reinterpret_cast<uint64_t*>(peers[size_t(g)]);
    }
    ML_CUDA_TRY(cudaMalloc(&d_peer_flags, sizeof(uint64_t*) * size_t(G)));
    ML_CUDA_TRY(cudaMemcpy(d_peer_flags, flags.data(), sizeof(uint64_t*) * size_t(G), cudaMemcpyHostToDevice));
    // every rank mapped every region before the first store into one
    return nccl_barrier(s);
  }
  mlStatus peer_barrier(cudaStream_t s) override {
    ++epoch;
    p2p_barrier_kernel<<<1, 32, 0, s>>>(d_peer_flags, reinterpret_cast<uint64_t*>(region), G, rank, epoch);
    ML_CUDA_TRY(cudaGetLastError());
    timing_mark("p2p_barrier", s);
    return ML_OK;
  }
  mlStatus all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    ML_NCCL_TRY(nccl().allGather(send, recv, bytes, ncclUint8, comm, s));
    timing_mark("nccl_all_gather", s);
    return ML_OK;
  }
  mlStatus all_to_all(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    ML_NCCL_TRY(nccl().groupStart());
    for (int g = 0; g < G; ++g) {
      ML_NCCL_TRY(nccl().send(static_cast<const char*>(send) + g * bytes, bytes, ncclUint8, g, comm, s));
      ML_NCCL_TRY(nccl().recv(static_cast<char*>(recv) + g * bytes, bytes, ncclUint8, g, comm, s));
    }
    ML_NCCL_TRY(nccl().groupEnd());
    timing_mark("nccl_all_to_all", s);
    return ML_OK;
  }
  mlStatus reduce_scatter_f32(const float* send, float* recv, size_t count, cudaStream_t s) override {
    ML_NCCL_TRY(nccl().reduceScatter(send, recv, count, ncclFloat32, ncclSum, comm, s));
    timing_mark("nccl_reduce_scatter", s);
    return ML_OK;
  }
  bool has_p2p() const override { return true; }
  mlStatus sendrecv(const void* send, int to, void* recv, int from, size_t bytes,
                    cudaStream_t s) override {
    ML_NCCL_TRY(nccl().groupStart());
    ML_NCCL_TRY(nccl().send(send, bytes, ncclUint8, to, comm, s));
    ML_NCCL_TRY(nccl().recv(recv, bytes, ncclUint8, from, comm, s));
    ML_NCCL_TRY(nccl().groupEnd());
    timing_mark("nccl_sendrecv", s);
    return ML_OK;
  }
};

__global__ void add_f32_kernel(float* dst, const float* src, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] += src[i];
}

// G ranks as host threads of one process on one device.  Each collective:
// the caller's stream is drained, every rank publishes its buffers, a
// barrier, each rank copies what it receives (in rank order), a barrier.
struct Hub {
  int G;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> send;
  explicit Hub(int g) : G(g), send(size_t(g), nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t my = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my; });
    }
  }
};

struct HubTransport : Transport {
  Hub* hub = nullptr;
  // peer memory of G threads on one device: plain device pointers, the
  // barrier a host one after draining the stream (no kernel ever waits on
  // another rank's kernel)
  bool peer_on = false;
  char* region = nullptr;
  size_t region_bytes = 0;
  std::vector<char*> peers;
  ~HubTransport() override {
    if (region) cudaFree(region);
  }
  bool has_peer_mem() const override { return peer_on && G > 1; }
  char* peer_region(int g) override { return peers[size_t(g)]; }
  mlStatus peer_setup(size_t bytes, cudaStream_t s) override {
    if (bytes <= region_bytes) return ML_OK;
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    hub->barrier();                        // nobody still uses the old regions
    if (region) cudaFree(region);
    ML_CUDA_TRY(cudaMalloc(&region, bytes));
    region_bytes = bytes;
    hub->send[size_t(rank)] = region;
    hub->barrier();
    peers.assign(size_t(G), nullptr);
    for (int g = 0; g < G; ++g) peers[size_t(g)] = static_cast<char*>(const_cast<void*>(hub->send[size_t(g)]));
    hub->barrier();
    return ML_OK;
  }
  mlStatus peer_barrier(cudaStream_t s) override {
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    hub->barrier();
    return ML_OK;
  }
  mlStatus publish(const void* p, cudaStream_t s) {
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    hub->send[size_t(rank)] = p;
    hub->barrier();
    return ML_OK;
  }
  mlStatus done(cudaStream_t s) {
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    hub->barrier();
    return ML_OK;
  }
  mlStatus all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    ML_TRY(publish(send, s));
    for (int g = 0; g < G; ++g)
      ML_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + g * bytes, hub->send[size_t(g)], bytes,
                                  cudaMemcpyDeviceToDevice, s));
    return done(s);
  }
  mlStatus all_to_all(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    ML_TRY(publish(send, s));
    for (int g = 0; g < G; ++g)
      ML_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(recv) + g * bytes,
                                  static_cast<const char*>(hub->send[size_t(g)]) + size_t(rank) * bytes,
                                  bytes, cudaMemcpyDeviceToDevice, s));
    return done(s);
  }
  mlStatus reduce_scatter_f32(const float* send, float* recv, size_t count, cudaStream_t s) override {
    ML_TRY(publish(send, s));
    ML_CUDA_TRY(cudaMemcpyAsync(recv, static_cast<const float*>(hub->send[0]) + size_t(rank) * count,
                                count * sizeof(float), cudaMemcpyDeviceToDevice, s));
    for (int g = 1; g < G; ++g) {     // fixed order -> deterministic
      add_f32_kernel<<<256, 256, 0, s>>>(recv, static_cast<const float*>(hub->send[size_t(g)]) +
                                                   size_t(rank) * count, int64_t(count));
      ML_LAUNCH_CHECK("group_hub_add");
    }
    return done(s);
  }
};

// One rank of a G-rank group with the network removed (t_ref(G)
// = this rank's work with the collectives replaced by local copies), running
// exactly the group's code path on one GPU.  An all-gather copies this rank's
// chunk into place and the other ranks' chunks from a caller capture: the
// next capture (cyclically) whose size is G x the chunk -- per step: the
// packed (idx, w), then the sorted lists of the inverse map; without a match
// the own chunk is replicated.  Every other exchange moves this rank's own
// data (shapes right; values do not change the work).
struct LoopbackTransport : Transport {
  std::vector<const char*> src;
  std::vector<size_t> src_bytes;
  size_t next = 0;
  mlStatus all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    const char* from = nullptr;
    for (size_t k = 0; k < src.size() && !from; ++k) {
      const size_t c = (next + k) % src.size();
      if (src_bytes[c] == size_t(G) * bytes) {
        from = src[c];
        next = c + 1;
      }
    }
    char* r = static_cast<char*>(recv);
    for (int g = 0; g < G; ++g) {
      const void* piece = (g == rank || !from) ? send : static_cast<const void*>(from + size_t(g) * bytes);
      if (piece != r + size_t(g) * bytes)
        ML_CUDA_TRY(cudaMemcpyAsync(r + size_t(g) * bytes, piece, bytes, cudaMemcpyDeviceToDevice, s));
    }
    timing_mark("loopback_all_gather", s);
    return ML_OK;
  }
  mlStatus all_to_all(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    ML_CUDA_TRY(cudaMemcpyAsync(recv, send, size_t(G) * bytes, cudaMemcpyDeviceToDevice, s));
    timing_mark("loopback_all_to_all", s);
    return ML_OK;
  }
  mlStatus reduce_scatter_f32(const float* send, float* recv, size_t count, cudaStream_t s) override {
    ML_CUDA_TRY(cudaMemcpyAsync(recv, send + size_t(rank) * count, count * sizeof(float),
                                cudaMemcpyDeviceToDevice, s));
    timing_mark("loopback_reduce_scatter", s);
    return ML_OK;
  }
  bool has_p2p() const override { return true; }
  mlStatus sendrecv(const void* send, int, void* recv, int, size_t bytes, cudaStream_t s) override {
    ML_CUDA_TRY(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
    timing_mark("loopback_sendrecv", s);
    return ML_OK;
  }
  // fused exchange: every "peer" region is a local buffer of its own (the
  // stores cost the HBM bytes the NVLink stores would not), no barrier
  bool peer_on = false;
  std::vector<char*> regions;
  size_t region_bytes = 0;
  ~LoopbackTransport() override {
    for (char* p : regions) cudaFree(p);
  }
  bool has_peer_mem() const override { return peer_on && G > 1; }
  char* peer_region(int g) override { return regions[size_t(g)]; }
  mlStatus peer_setup(size_t bytes, cudaStream_t s) override {
    if (bytes <= region_bytes) return ML_OK;
    ML_CUDA_TRY(cudaStreamSynchronize(s));
    for (char* p : regions) cudaFree(p);
    regions.assign(size_t(G), nullptr);
    for (auto& p : regions) ML_CUDA_TRY(cudaMalloc(&p, bytes));
    region_bytes = bytes;
    return ML_OK;
  }
  mlStatus peer_barrier(cudaStream_t) override { return ML_OK; }
};

// ------------------------------------------------------------ layout kernels
// (idx, w) of T rows of B -> one packed [T][2B] int32 block (w as bits)
__global__ void pack_iw_kernel(const int32_t* idx, const float* w, int64_t T, int B, int32_t* out) {
  const int64_t n = T * B;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / B, j = i - t * B;
    out[t * 2 * B + j] = idx[i];
    out[t * 2 * B + B + j] = __float_as_int(w[i]);
  }
}
__global__ void unpack_iw_kernel(const int32_t* in, int64_t T, int B, int32_t* idx, float* w) {
  const int64_t n = T * B;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / B, j = i - t * B;
    idx[i] = in[t * 2 * B + j];
    w[i] = __int_as_float(in[t * 2 * B + B + j]);
  }
}

unsigned grid_for(int64_t n) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8)));
}

}  // namespace
}  // namespace ml

using namespace ml;

// ------------------------------------------------------------ the group
struct mlGroup_ {
  Transport* tr = nullptr;
  int device = 0;
  cudaStream_t comm = nullptr, aux = nullptr, prep = nullptr;
  cudaEvent_t ev[8] = {};
  std::vector<cudaEvent_t> blk;     // per-block events of the pipelined forward
  cudaEvent_t state_ready = nullptr;
  uint64_t p2p_steps = 0;           // fused forward exchanges so far (double-buffer parity)
  uint64_t p2p_bwd_steps = 0;       // fused backward exchanges so far
};

namespace ml {
namespace {

// ML_GROUP_P2P=1: the fused peer-memory forward exchange by default (else
// ml_group_set_p2p)
bool p2p_env() {
  const char* e = std::getenv("ML_GROUP_P2P");
  return e && e[0] == '1';
}

mlStatus group_make(mlGroup_* g) {
  ML_CUDA_TRY(cudaGetDevice(&g->device));
  int lo = 0, hi = 0;
  ML_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  ML_CUDA_TRY(cudaStreamCreateWithPriority(&g->comm, cudaStreamNonBlocking, hi));
  ML_CUDA_TRY(cudaStreamCreateWithFlags(&g->aux, cudaStreamNonBlocking));
  ML_CUDA_TRY(cudaStreamCreateWithFlags(&g->prep, cudaStreamNonBlocking));
  for (auto& e : g->ev) ML_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  g->blk.resize(size_t(g->tr->G));
  for (auto& e : g->blk) ML_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  ML_CUDA_TRY(cudaEventCreateWithFlags(&g->state_ready, cudaEventDisableTiming));
  return ML_OK;
}

mlStatus dep(cudaStream_t from, cudaStream_t to, cudaEvent_t e) {
  ML_CUDA_TRY(cudaEventRecord(e, from));
  ML_CUDA_TRY(cudaStreamWaitEvent(to, e, 0));
  return ML_OK;
}

mlStatus check_group_shape(const mlGroup_* g, const mlBagShape* s, mlOutMode mode) {
  if (!g || !g->tr) return fail(ML_ERR_ARG, "null group");
  if (!s) return fail(ML_ERR_ARG, "null shape");
  if (mode != ML_OUT_ALLTOALL && mode != ML_OUT_ALLGATHER) return fail(ML_ERR_ARG, "unknown output mode");
  const int G = g->tr->G;
  if (s->dv % G) return fail(ML_ERR_CONFIG, "group: G must divide dv (SPEC S:401)");
  if ((int64_t(s->dv / G) * int64_t(dtype_size(s->dtype))) % 16)
    return fail(ML_ERR_CONFIG, "group: (dv/G)*e must be a multiple of 16 bytes");
  if (int64_t(G) * s->T * s->B >= (int64_t(1) << 31)) return fail(ML_ERR_CONFIG, "group: G*T*B must be < 2^31");
  return ML_OK;
}

// the local bag over all group tokens on the [N, dv/G] shard
mlBagShape shard_shape(const mlGroup_* g, const mlBagShape& s) {
  mlBagShape b = s;
  b.dv = s.dv / g->tr->G;
  b.T = s.T * g->tr->G;
  return b;
}

// The exchange region of the fused (peer-memory) form, identical on every
// rank for a shape: epoch flags, then the forward's y blocks, the backward's
// dy blocks and partial dw blocks -- each section double-buffered by the
// parity of its exchange count (a half is rewritten two exchanges later,
// after the barrier of the one in between, which its receiver passes only
// after consuming it).
struct PeerLayout { size_t y_off, y_half, dy_off, dy_half, dw_off, dw_half, dw_blk, total; };
PeerLayout peer_layout(const mlGroup_* g, const mlBagShape& s) {
  const int G = g->tr->G;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t blk = size_t(s.T) * (s.dv / G) * dtype_size(s.dtype);
  PeerLayout L;
  L.y_half = up(size_t(G) * blk);
  L.dy_half = L.y_half;
  L.dw_blk = size_t(s.T) * s.B * sizeof(float);
  L.dw_half = up(size_t(G) * L.dw_blk);
  L.y_off = kPeerFlagBytes;
  L.dy_off = L.y_off + 2 * L.y_half;
  L.dw_off = L.dy_off + 2 * L.dy_half;
  L.total = L.dw_off + 2 * L.dw_half;
  return L;
}

struct FwdBufs { int32_t* iw_send; int32_t* iw_recv; void* y_part; void* recv; };
void fwd_carve(Carver& c, const mlGroup_* g, const mlBagShape& s, mlOutMode mode, FwdBufs& b) {
  const int G = g->tr->G;
  const int64_t e = int64_t(dtype_size(s.dtype));
  const int64_t slice = int64_t(s.T) * (s.dv / G);   // one block of one slice
  b.iw_send = c.take<int32_t>(int64_t(s.T) * 2 * s.B);
  b.iw_recv = c.take<int32_t>(int64_t(G) * s.T * 2 * s.B);
  b.y_part = c.take<char>(int64_t(G) * slice * e);
  b.recv = c.take<char>((mode == ML_OUT_ALLGATHER ? int64_t(G) * G : int64_t(G)) * slice * e);
}

// (idx, w) all-gather: the caller's [T_loc, B] -> idx_all / w_all [G*T_loc, B]
mlStatus gather_iw(mlGroup_* g, const mlBagShape& s, const int32_t* idx, const float* w,
                   int32_t* idx_all, float* w_all, FwdBufs& b, cudaStream_t st) {
  const int G = g->tr->G;
  const int64_t n = int64_t(s.T) * s.B;
  pack_iw_kernel<<<grid_for(n), 256, 0, st>>>(idx, w, s.T, s.B, b.iw_send);
  count_launch();
  ML_CUDA_TRY(cudaGetLastError());
  ML_TRY(g->tr->all_gather(b.iw_send, b.iw_recv, size_t(n) * 2 * sizeof(int32_t), st));
  unpack_iw_kernel<<<grid_for(n * G), 256, 0, st>>>(b.iw_recv, int64_t(s.T) * G, s.B, idx_all, w_all);
  count_launch();
  ML_CUDA_TRY(cudaGetLastError());
  return ML_OK;
}

// the bag forward block by block, each finished block leaving on the
// communication stream while the next one is computed.  Mode P: block of
// rank `to` goes to `to` (ring step i: to = rank+1+i, from = rank-1-i; own
// block last); recv [G][T_loc][dv/G] from every rank.  Mode N: blocks in rank
// order, each all-gathered: recv [block][G src][T_loc][dv/G].
mlStatus bag_blocks(mlGroup_* g, const mlBagShape& s, mlOutMode mode, const void* V_shard,
                    const int32_t* idx_all, const float* w_all, FwdBufs& b, cudaStream_t st,
                    const void** recv_out) {
  const int G = g->tr->G, r = g->tr->rank;
  const int dvG = s.dv / G;
  const int64_t e = int64_t(dtype_size(s.dtype));
  const size_t blk_bytes = size_t(s.T) * dvG * e;
  const mlBagShape bs{s.N, dvG, s.T, s.B, s.dtype, ML_F32};
  *recv_out = b.recv;
  if (mode == ML_OUT_ALLTOALL && g->tr->has_peer_mem()) {
    // Fused exchange (peer memory): the bag kernel of block `to` stores its
    // output rows straight into rank `to`'s exchange region, slot `r`, over
    // NVLink -- the transfer rides inside the HBM-bound gather, no separate
    // collective.  Regions are double-buffered by step parity: a writer
    // reuses a half only two steps later, after the barrier of the step in
    // between, which the receiver passes only after unpacking this one.
    const PeerLayout L = peer_layout(g, s);
    ML_TRY(g->tr->peer_setup(L.total, st));
    const size_t off = L.y_off + size_t(g->p2p_steps & 1) * L.y_half;
    ++g->p2p_steps;
    // ONE bag launch over all G*T_loc tokens: token block `to` (rank `to`'s
    // tokens) is stored into rank `to`'s region, slot `r`
    void* blocks[kMaxOutBlocks];
    if (G > kMaxOutBlocks) return fail(ML_ERR_CONFIG, "fused exchange: G <= 64");
    for (int to = 0; to < G; ++to) blocks[to] = g->tr->peer_region(to) + off + size_t(r) * blk_bytes;
    BagFwdArgs a;
    a.V = V_shard; a.ldv = dvG; a.N = s.N;
    a.idx = idx_all; a.w = w_all; a.B = s.B; a.nbags = G * s.T; a.dv = dvG;
    a.out = blocks[0]; a.ldo = dvG; a.dtype = s.dtype;
    a.out_blocks = blocks; a.block_rows = s.T;
    a.name = "embbag_fwd";
    timing_mark(nullptr, st);
    ML_TRY(launch_bag_fwd(a, st));
    ML_TRY(g->tr->peer_barrier(st));
    *recv_out = g->tr->peer_region(r) + off;
    return ML_OK;
  }
  // Mode P: one bag launch over all G*T_loc tokens, then one all-to-all --
  // measured faster than the block pipeline (one launch per destination's
  // T_loc tokens, each block sent while the next is gathered): a block fills
  // less than half the GPU at C4/C5 (the launches cost 0.08-0.13 ms more per
  // step than the NVLink transfer they would hide, 10-80 us at 700 GB/s).
  // ML_GROUP_PIPELINE=1 restores the pipeline.
  static const bool pipe_env = [] {
    const char* e = std::getenv("ML_GROUP_PIPELINE");
    return e && e[0] == '1';
  }();
  const bool p2p = mode == ML_OUT_ALLTOALL && g->tr->has_p2p() && pipe_env;
  const bool pipelined = p2p || mode == ML_OUT_ALLGATHER;
  if (mode == ML_OUT_ALLTOALL && !pipelined) {
    const mlBagShape all{s.N, dvG, G * s.T, s.B, s.dtype, ML_F32};
    ML_TRY((embbag_fwd(&all, V_shard, idx_all, w_all, nullptr, b.y_part, nullptr, st)));
    return g->tr->all_to_all(b.y_part, b.recv, blk_bytes, st);
  }
  // measurement mode (ml_set_serial): the exchange runs on the caller's
  // stream, so each collective's timing event brackets it alone
  cudaStream_t cs = serial_mode() ? st : g->comm;
  if (pipelined) ML_TRY(dep(st, cs, g->ev[0]));    // inputs of the exchange are ready
  for (int i = 0; i < G; ++i) {
    const int blk = mode == ML_OUT_ALLTOALL ? (r + 1 + i) % G : i;
    char* yp = static_cast<char*>(b.y_part) + size_t(blk) * blk_bytes;
    ML_TRY((embbag_fwd(&bs, V_shard, idx_all + int64_t(blk) * s.T * s.B,
                                   w_all + int64_t(blk) * s.T * s.B, nullptr, yp, nullptr, st)));
    if (!pipelined) continue;
    ML_CUDA_TRY(cudaEventRecord(g->blk[size_t(i)], st));
    ML_CUDA_TRY(cudaStreamWaitEvent(cs, g->blk[size_t(i)], 0));
    if (p2p) {
      const int from = ((r - 1 - i) % G + G) % G;
      ML_TRY(g->tr->sendrecv(yp, blk, static_cast<char*>(b.recv) + size_t(from) * blk_bytes, from,
                             blk_bytes, cs));
    } else {
      ML_TRY(g->tr->all_gather(yp, static_cast<char*>(b.recv) + size_t(blk) * G * blk_bytes,
                               blk_bytes, cs));
    }
  }
  if (pipelined) return dep(cs, st, g->ev[1]);
  return g->tr->all_to_all(b.y_part, b.recv, blk_bytes, st);
}

// The group's backward state: the bag-level state of
// the shard shape (the merged inverse map of all G*T_loc tokens) followed by
// this rank's sorted list, the G gathered lists and the local sort's
// workspace.  Built once per group: each rank sorts only its own positions,
// the sorted lists are all-gathered and merged (merge.cu), instead of every
// rank sorting all G*T_loc*B positions.
struct GroupState { void* bag; size_t bag_bytes; int32_t* send; int32_t* recv; void* sort_ws; size_t sort_bytes; };
mlStatus group_state_carve(Carver& c, const mlGroup_* g, const mlBagShape& s, GroupState& gs) {
  const mlBagShape bs = shard_shape(g, s);
  const int64_t P_loc = int64_t(s.T) * s.B;
  ML_TRY((embbag_bwd_state_bytes(&bs, &gs.bag_bytes)));
  ML_TRY((embbag_bwd_group_sort_local_workspace(&s, &gs.sort_bytes)));
  gs.bag = c.take<char>(int64_t(gs.bag_bytes));
  gs.send = c.take<int32_t>(2 * P_loc);
  gs.recv = c.take<int32_t>(int64_t(g->tr->G) * 2 * P_loc);
  gs.sort_ws = c.take<char>(int64_t(gs.sort_bytes));
  return ML_OK;
}

// phase A (preparation stream): sort this rank's own positions
mlStatus group_state_local(mlGroup_* g, const mlBagShape& s, const int32_t* idx_own, GroupState& gs,
                           cudaStream_t st) {
  cudaStream_t ps = serial_mode() ? st : g->prep;
  ML_TRY(dep(st, ps, g->ev[2]));
  ML_TRY((embbag_bwd_group_sort_local(&s, g->tr->rank, idx_own, gs.send, gs.sort_ws, gs.sort_bytes, ps)));
  return ML_OK;
}

// phase B: the lists' all-gather on the communication stream, then the merge
// and the run table on the preparation stream -> state_ready
mlStatus group_state_merge(mlGroup_* g, const mlBagShape& s, GroupState& gs, cudaStream_t st) {
  cudaStream_t ps = serial_mode() ? st : g->prep;
  cudaStream_t cs = serial_mode() ? st : g->comm;
  const int64_t P_loc = int64_t(s.T) * s.B;
  // after the local sort AND after every collective already issued on the
  // caller's stream (one device order for all of the group's NCCL calls)
  ML_TRY(dep(ps, cs, g->ev[7]));
  if (cs != st) ML_TRY(dep(st, cs, g->ev[5]));
  ML_TRY(g->tr->all_gather(gs.send, gs.recv, size_t(2 * P_loc) * sizeof(int32_t), cs));
  ML_TRY(dep(cs, ps, g->ev[7]));
  const mlBagShape bs = shard_shape(g, s);
  ML_TRY((embbag_bwd_group_merge(&bs, g->tr->G, gs.recv, gs.bag, gs.bag_bytes, ps)));
  ML_CUDA_TRY(cudaEventRecord(g->state_ready, ps));
  return ML_OK;
}

}  // namespace
}  // namespace ml

extern "C" {

mlStatus ml_group_unique_id(void* id) {
  ML_API_BEGIN_X
  if (!id) return fail(ML_ERR_ARG, "null id");
  if (!nccl().ok) return fail(ML_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId u;
  ML_NCCL_TRY(nccl().getUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return ML_OK;
  ML_API_END_X
}

mlStatus ml_group_init(const void* id, int G, int rank, mlGroup* out) {
  ML_API_BEGIN_X
  if (!id || !out) return fail(ML_ERR_ARG, "null argument");
  if (G < 1 || rank < 0 || rank >= G) return fail(ML_ERR_CONFIG, "group: need 0 <= rank < G");
  if (!nccl().ok) return fail(ML_ERR_NCCL, "libnccl.so.2 not found");
  auto* t = new NcclTransport();
  t->G = G;
  t->rank = rank;
  t->peer_on = p2p_env();
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  const ncclResult_t r = nccl().commInitRank(&t->comm, G, u, rank);
  if (r != ncclSuccess) {
    delete t;
    return fail(ML_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().errorString(r));
  }
  auto* g = new mlGroup_();
  g->tr = t;
  const mlStatus st = group_make(g);
  if (st != ML_OK) return st;
  *out = g;
  return ML_OK;
  ML_API_END_X
}

mlStatus ml_group_hub_create(int G, void** hub) {
  ML_API_BEGIN_X
  if (!hub || G < 1) return fail(ML_ERR_ARG, "hub: need G >= 1");
  *hub = new Hub(G);
  return ML_OK;
  ML_API_END_X
}

mlStatus ml_group_hub_destroy(void* hub) {
  delete static_cast<Hub*>(hub);
  return ML_OK;
}

mlStatus ml_group_init_hub(void* hub, int rank, mlGroup* out) {
  ML_API_BEGIN_X
  if (!hub || !out) return fail(ML_ERR_ARG, "null argument");
  Hub* h = static_cast<Hub*>(hub);
  if (rank < 0 || rank >= h->G) return fail(ML_ERR_CONFIG, "group: need 0 <= rank < G");
  auto* t = new HubTransport();
  t->G = h->G;
  t->rank = rank;
  t->peer_on = p2p_env();
  t->hub = h;
  auto* g = new mlGroup_();
  g->tr = t;
  ML_TRY(group_make(g));
  *out = g;
  return ML_OK;
  ML_API_END_X
}

mlStatus ml_group_init_loopback(int G, int rank, const void* const* sources, const size_t* bytes,
                                int n_sources, mlGroup* out) {
  ML_API_BEGIN_X
  if (!out) return fail(ML_ERR_ARG, "null argument");
  if (G < 1 || rank < 0 || rank >= G) return fail(ML_ERR_CONFIG, "group: need 0 <= rank < G");
  if (n_sources < 0 || (n_sources > 0 && (!sources || !bytes))) return fail(ML_ERR_ARG, "bad sources");
  auto* t = new LoopbackTransport();
  t->G = G;
  t->rank = rank;
  for (int k = 0; k < n_sources; ++k) {
    t->src.push_back(static_cast<const char*>(sources[k]));
    t->src_bytes.push_back(bytes[k]);
  }
  auto* g = new mlGroup_();
  g->tr = t;
  ML_TRY(group_make(g));
  *out = g;
  return ML_OK;
  ML_API_END_X
}

mlStatus ml_group_destroy(mlGroup g) {
  ML_API_BEGIN_X
  if (!g) return ML_OK;
  cudaStreamSynchronize(g->comm);
  cudaStreamSynchronize(g->aux);
  cudaStreamSynchronize(g->prep);
  for (auto e : g->ev) cudaEventDestroy(e);
  for (auto e : g->blk) cudaEventDestroy(e);
  cudaEventDestroy(g->state_ready);
  cudaStreamDestroy(g->comm);
  cudaStreamDestroy(g->aux);
  cudaStreamDestroy(g->prep);
  delete g->tr;
  delete g;
  return ML_OK;
  ML_API_END_X
}

mlStatus ml_group_set_p2p(mlGroup g, int on) {
  ML_API_BEGIN_X
  if (!g) return fail(ML_ERR_ARG, "null group");
  if (auto* t = dynamic_cast<NcclTransport*>(g->tr)) t->peer_on = on != 0;
  else if (auto* h = dynamic_cast<HubTransport*>(g->tr)) h->peer_on = on != 0;
  else if (auto* l = dynamic_cast<LoopbackTransport*>(g->tr)) l->peer_on = on != 0;
  return ML_OK;
  ML_API_END_X
}

mlStatus ml_group_info(mlGroup g, int* G, int* rank) {
  if (!g) return fail(ML_ERR_ARG, "null group");
  if (G) *G = g->tr->G;
  if (rank) *rank = g->tr->rank;
  return ML_OK;
}

// ------------------------------------------------------------ bag level
mlStatus embbag_fwd_group_workspace(mlGroup g, const mlBagShape* shape, mlOutMode mode, size_t* bytes) {
  ML_API_BEGIN_X
  ML_TRY(check_group_shape(g, shape, mode));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  FwdBufs b;
  fwd_carve(c, g, *shape, mode, b);
  *bytes = c.used;
  return ML_OK;
  ML_API_END_X
}

mlStatus embbag_fwd_group(mlGroup g, const mlBagShape* shape, const void* V_shard,
                          const int32_t* idx_local, const float* w_local, int32_t* idx_all,
                          float* w_all, mlOutMode mode, void* y, void* ws, size_t ws_bytes,
                          void* stream) {
  ML_API_BEGIN_X
  ML_TRY(check_group_shape(g, shape, mode));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = g->tr->G;
  if (shape->T == 0) return ML_OK;
  if (!V_shard || !idx_local || !w_local || !idx_all || !w_all || !y || !ws)
    return fail(ML_ERR_ARG, "null pointer argument");
  size_t need = 0;
  ML_TRY(embbag_fwd_group_workspace(g, shape, mode, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_fwd_group: workspace too small");
  Carver c(ws);
  FwdBufs b;
  fwd_carve(c, g, *shape, mode, b);
  ML_TRY(gather_iw(g, *shape, idx_local, w_local, idx_all, w_all, b, st));
  const void* recv = nullptr;
  ML_TRY(bag_blocks(g, *shape, mode, V_shard, idx_all, w_all, b, st, &recv));
  const size_t blk_bytes = size_t(shape->T) * (shape->dv / G) * dtype_size(shape->dtype);
  if (mode == ML_OUT_ALLTOALL)
    return ml_group_unpack(recv, G, shape->T, shape->dv, nullptr, y, nullptr, shape->dtype, st);
  for (int blk = 0; blk < G; ++blk)
    ML_TRY((ml_group_unpack(static_cast<char*>(b.recv) + size_t(blk) * G * blk_bytes, G,
                                        shape->T, shape->dv, nullptr,
                                        static_cast<char*>(y) + size_t(blk) * G * blk_bytes, nullptr,
                                        shape->dtype, st)));
  return ML_OK;
  ML_API_END_X
}

struct BwdGroupBufs { void* dy_send; void* dy_recv; float* dw_part; void* state; void* bag_ws; };
static mlStatus bwd_carve(Carver& c, const mlGroup_* g, const mlBagShape& s, BwdGroupBufs& b,
                          bool own_state) {
  const int G = g->tr->G;
  const int64_t e = int64_t(dtype_size(s.dtype));
  const mlBagShape bs = shard_shape(g, s);
  b.dy_send = c.take<char>(int64_t(s.T) * s.dv * e);
  b.dy_recv = c.take<char>(int64_t(G) * s.T * (s.dv / G) * e);
  b.dw_part = c.take<float>(int64_t(G) * s.T * s.B);
  size_t sb = 0, wb = 0;
  ML_TRY((embbag_bwd_state_bytes(&bs, &sb)));
  ML_TRY((embbag_bwd_workspace(&bs, &wb)));
  b.state = own_state ? c.take<char>(sb) : nullptr;
  b.bag_ws = c.take<char>(wb);
  return ML_OK;
}

mlStatus embbag_bwd_group_workspace(mlGroup g, const mlBagShape* shape, mlOutMode mode, size_t* bytes) {
  ML_API_BEGIN_X
  ML_TRY(check_group_shape(g, shape, mode));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  BwdGroupBufs b;
  ML_TRY(bwd_carve(c, g, *shape, b, true));
  *bytes = c.used;
  return ML_OK;
  ML_API_END_X
}

mlStatus embbag_bwd_group_state_bytes(mlGroup g, const mlBagShape* shape, size_t* bytes) {
  ML_API_BEGIN_X
  ML_TRY(check_group_shape(g, shape, ML_OUT_ALLTOALL));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  GroupState gs;
  ML_TRY(group_state_carve(c, g, *shape, gs));
  *bytes = c.used;
  return ML_OK;
  ML_API_END_X
}

mlStatus embbag_bwd_group(mlGroup g, const mlBagShape* shape, const void* V_shard,
                          const int32_t* idx_all, const float* w_all, const void* dy,
                          mlOutMode mode, const void* state, size_t state_bytes, int32_t* rows,
                          void* dV_shard, int32_t* U, float* dw_local, void* ws, size_t ws_bytes,
                          void* stream) {
  ML_API_BEGIN_X
  ML_TRY(check_group_shape(g, shape, mode));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = g->tr->G, r = g->tr->rank;
  if (!U) return fail(ML_ERR_ARG, "null U");
  if (shape->T == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), st));
    return ML_OK;
  }
  if (!V_shard || !idx_all || !w_all || !dy || !rows || !dV_shard || !dw_local || !ws)
    return fail(ML_ERR_ARG, "null pointer argument");
  size_t need = 0;
  ML_TRY(embbag_bwd_group_workspace(g, shape, mode, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_bwd_group: workspace too small");
  Carver c(ws);
  BwdGroupBufs b;
  ML_TRY(bwd_carve(c, g, *shape, b, true));
  const mlBagShape bs = shard_shape(g, *shape);
  const int dvG = shape->dv / G;
  const size_t e = dtype_size(shape->dtype);
  size_t wb = 0, sb = 0;
  ML_TRY((embbag_bwd_workspace(&bs, &wb)));
  ML_TRY((embbag_bwd_state_bytes(&bs, &sb)));
  // the state's list all-gather ran on the communication stream: wait for the
  // state BEFORE this call's collectives, so that every NCCL operation of the
  // group is ordered on the device exactly as it was issued (no two in flight
  // on different streams)
  if (state) {
    if (state_bytes < sb) return fail(ML_ERR_WORKSPACE, "embbag_bwd_group: state too small");
    ML_CUDA_TRY(cudaStreamWaitEvent(st, g->state_ready, 0));
  }
  const bool fused = g->tr->has_peer_mem();
  PeerLayout L{};
  size_t par = 0;
  const void* dy_slices = b.dy_recv;
  if (fused) {   // fused exchange: stores straight into the owners' regions
    L = peer_layout(g, *shape);
    ML_TRY(g->tr->peer_setup(L.total, st));
    par = size_t(g->p2p_bwd_steps++ & 1);
  }
  if (mode == ML_OUT_ALLTOALL && fused) {
    // slice g of this rank's dy rows -> rank g's region, slot r
    void* dst[kMaxOutBlocks];
    const size_t blk = size_t(shape->T) * dvG * e;
    for (int to = 0; to < G; ++to) dst[to] = g->tr->peer_region(to) + L.dy_off + par * L.dy_half + size_t(r) * blk;
    ML_TRY(launch_group_pack_peers(dy, G, shape->T, dvG, dst, shape->dtype, st));
    ML_TRY(g->tr->peer_barrier(st));
    dy_slices = g->tr->peer_region(r) + L.dy_off + par * L.dy_half;
  } else if (mode == ML_OUT_ALLTOALL) {
    // dy of this rank's tokens -> [G][T_loc][dv/G] -> slice g to rank g
    ML_TRY((ml_group_pack(dy, G, shape->T, shape->dv, b.dy_send, shape->dtype, st)));
    ML_TRY(g->tr->all_to_all(b.dy_send, b.dy_recv, size_t(shape->T) * dvG * e, st));
  } else {
    // dy replicated [G*T_loc, dv]: this rank's column slice
    ML_CUDA_TRY(cudaMemcpy2DAsync(b.dy_recv, size_t(dvG) * e, static_cast<const char*>(dy) + size_t(r) * dvG * e,
                                  size_t(shape->dv) * e, size_t(dvG) * e, size_t(G) * shape->T,
                                  cudaMemcpyDeviceToDevice, st));
  }
  if (!state) {
    ML_TRY((embbag_bwd_prepare(&bs, idx_all, b.state, sb, st)));
    state = b.state;
  }
  ML_TRY((embbag_bwd_state(&bs, V_shard, w_all, dy_slices, state, sb, rows, dV_shard, U,
                                       b.dw_part, b.bag_ws, wb, st)));
  // partial dw (a dot over this rank's dv/G columns) summed over the shards
  if (fused) {   // block g -> rank g's region slot r; the owner sums the G slots in rank order
    const int64_t n = int64_t(shape->T) * shape->B;
    for (int to = 0; to < G; ++to)
      ML_CUDA_TRY(cudaMemcpyAsync(g->tr->peer_region(to) + L.dw_off + par * L.dw_half + size_t(r) * L.dw_blk,
                                  b.dw_part + int64_t(to) * n, L.dw_blk, cudaMemcpyDeviceToDevice, st));
    ML_TRY(g->tr->peer_barrier(st));
    return launch_sum_ranks(reinterpret_cast<const float*>(g->tr->peer_region(r) + L.dw_off + par * L.dw_half),
                            G, n, dw_local, st);
  }
  return g->tr->reduce_scatter_f32(b.dw_part, dw_local, size_t(shape->T) * shape->B, st);
  ML_API_END_X
}

// the backward's inverse index map of idx_all (a collective: every rank
// calls it): this rank's own positions sorted on the group's preparation
// stream, the G sorted lists all-gathered on the communication stream and
// merged (ordered after the caller's work so far); embbag_bwd_group /
// memory_layer_bwd_group wait for it
mlStatus embbag_bwd_group_prepare(mlGroup g, const mlBagShape* shape, const int32_t* idx_all,
                                  void* state, size_t state_bytes, void* stream) {
  ML_API_BEGIN_X
  ML_TRY(check_group_shape(g, shape, ML_OUT_ALLTOALL));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t need = 0;
  ML_TRY(embbag_bwd_group_state_bytes(g, shape, &need));
  if (!state || state_bytes < need) return fail(ML_ERR_WORKSPACE, "embbag_bwd_group_prepare: state too small");
  if (shape->T > 0 && !idx_all) return fail(ML_ERR_ARG, "null idx_all");
  Carver c(state);
  GroupState gs;
  ML_TRY(group_state_carve(c, g, *shape, gs));
  const int64_t P_loc = int64_t(shape->T) * shape->B;
  ML_TRY(group_state_local(g, *shape, idx_all + int64_t(g->tr->rank) * P_loc, gs, st));
  return group_state_merge(g, *shape, gs, st);
  ML_API_END_X
}

// ------------------------------------------------------------ layer level
static mlStatus check_layer_group(const mlGroup_* g, const mlLayerShape* s, mlOutMode mode) {
  if (!s) return fail(ML_ERR_ARG, "null shape");
  if (!s->gated) return fail(ML_ERR_UNSUPPORTED, "memory_layer_*_group: the gated (Memory+) layer only");
  const mlBagShape b{s->N, s->dv, s->pkm.T, s->pkm.H * s->pkm.k, s->pkm.dtype, s->grad_dtype};
  return check_group_shape(g, &b, mode);
}
static mlBagShape bag_of_layer(const mlLayerShape& s) {
  return mlBagShape{s.N, s.dv, s.pkm.T, s.pkm.H * s.pkm.k, s.pkm.dtype, s.grad_dtype};
}

struct LayerFwdGroupBufs { FwdBufs f; void* pkm_ws; size_t pkm_bytes; void* z; void* gemm_ws; };
static mlStatus layer_fwd_group_carve(Carver& c, const mlGroup_* g, const mlLayerShape& s,
                                      mlOutMode mode, LayerFwdGroupBufs& b) {
  fwd_carve(c, g, bag_of_layer(s), mode, b.f);
  ML_TRY((pkm_topk_workspace(&s.pkm, &b.pkm_bytes)));
  b.pkm_ws = c.take<char>(b.pkm_bytes);
  b.z = c.take<char>(int64_t(s.pkm.T) * s.dv * int64_t(dtype_size(s.pkm.dtype)));
  b.gemm_ws = c.take<char>(kGemmWs);
  return ML_OK;
}

mlStatus memory_layer_fwd_group_workspace(mlGroup g, const mlLayerShape* shape, mlOutMode mode,
                                          size_t* bytes) {
  ML_API_BEGIN_X
  ML_TRY(check_layer_group(g, shape, mode));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  LayerFwdGroupBufs b;
  ML_TRY(layer_fwd_group_carve(c, g, *shape, mode, b));
  *bytes = c.used;
  return ML_OK;
  ML_API_END_X
}

mlStatus memory_layer_fwd_group(mlGroup g, const mlLayerShape* shape, mlOutMode mode, const void* x,
                                const void* q, const void* K1, const void* K2, const void* V_shard,
                                const void* W1, const void* W2, void* out, int32_t* idx_saved,
                                float* w_saved, int32_t* idx_all, float* w_all, void* g_saved,
                                void* y_saved, void* y_all, void* state, size_t state_bytes,
                                void* ws, size_t ws_bytes, void* stream) {
  ML_API_BEGIN_X
  ML_TRY(check_layer_group(g, shape, mode));
  const mlLayerShape& s = *shape;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int G = g->tr->G, r = g->tr->rank;
  const int T = s.pkm.T;
  if (T == 0) return ML_OK;
  if (!x || !q || !K1 || !K2 || !V_shard || !W1 || !W2 || !out || !idx_saved || !w_saved ||
      !idx_all || !w_all || !g_saved || !y_saved || !ws)
    return fail(ML_ERR_ARG, "null pointer argument");
  if (mode == ML_OUT_ALLGATHER && !y_all) return fail(ML_ERR_ARG, "mode N needs y_all");
  size_t need = 0;
  ML_TRY(memory_layer_fwd_group_workspace(g, shape, mode, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "memory_layer_fwd_group: workspace too small");
  Carver c(ws);
  LayerFwdGroupBufs b;
  ML_TRY(layer_fwd_group_carve(c, g, s, mode, b));
  const mlBagShape bag = bag_of_layer(s);
  const mlDtype dt = s.pkm.dtype;
  // g = x W1 on the aux stream, concurrent with the lookup and the exchange
  cudaStream_t as = serial_mode() ? st : g->aux;
  ML_TRY(dep(st, as, g->ev[3]));
  ML_TRY((ml_gemm(0, 0, T, s.dv, s.D, x, s.D, W1, s.dv, g_saved, s.dv, dt, 0, b.gemm_ws,
                              kGemmWs, as)));
  // own tokens' product-key lookup, then the (idx, w) all-gather
  ML_TRY((pkm_topk(&s.pkm, q, K1, K2, idx_saved, w_saved, nullptr, b.pkm_ws, b.pkm_bytes, st)));
  // the backward's state: own positions sorted beside the exchange and the
  // bag forward, the sorted lists exchanged and merged after the blocks
  GroupState gs{};
  if (state) {
    size_t sneed = 0;
    ML_TRY(embbag_bwd_group_state_bytes(g, &bag, &sneed));
    if (state_bytes < sneed) return fail(ML_ERR_WORKSPACE, "memory_layer_fwd_group: state too small");
    Carver sc(state);
    ML_TRY(group_state_carve(sc, g, bag, gs));
    ML_TRY(group_state_local(g, bag, idx_saved, gs, st));
  }
  ML_TRY(gather_iw(g, bag, idx_saved, w_saved, idx_all, w_all, b.f, st));
  const void* recv = nullptr;
  ML_TRY(bag_blocks(g, bag, mode, V_shard, idx_all, w_all, b.f, st, &recv));
  if (state) ML_TRY(group_state_merge(g, bag, gs, st));
  ML_TRY(dep(as, st, g->ev[4]));                   // g ready
  const size_t blk_bytes = size_t(T) * (s.dv / G) * dtype_size(dt);
  const void* own = mode == ML_OUT_ALLTOALL ? recv
                                            : static_cast<const char*>(b.f.recv) + size_t(r) * G * blk_bytes;
  ML_TRY((ml_group_unpack(own, G, T, s.dv, g_saved, y_saved, b.z, dt, st)));
  if (mode == ML_OUT_ALLGATHER)
    for (int blk = 0; blk < G; ++blk)
      ML_TRY((ml_group_unpack(static_cast<char*>(b.f.recv) + size_t(blk) * G * blk_bytes, G, T,
                                          s.dv, nullptr, static_cast<char*>(y_all) + size_t(blk) * G * blk_bytes,
                                          nullptr, dt, st)));
  return ml_gemm(0, 0, T, s.D, s.dv, b.z, s.dv, W2, s.D, out, s.D, dt, 0, b.gemm_ws, kGemmWs, st);
  ML_API_END_X
}

struct LayerBwdGroupBufs {
  BwdGroupBufs bag; void *dz, *z, *dy, *dg, *gemm_ws, *gemm_ws2, *pkm_ws; size_t pkm_bytes;
  float* dw_local;
};
static mlStatus layer_bwd_group_carve(Carver& c, const mlGroup_* g, const mlLayerShape& s,
                                      LayerBwdGroupBufs& b) {
  const int64_t act = int64_t(s.pkm.T) * s.dv * int64_t(dtype_size(s.pkm.dtype));
  ML_TRY(bwd_carve(c, g, bag_of_layer(s), b.bag, true));
  b.dz = c.take<char>(act);
  b.z = c.take<char>(act);
  b.dy = c.take<char>(act);
  b.dg = c.take<char>(act);
  b.gemm_ws = c.take<char>(kGemmWs);
  b.gemm_ws2 = c.take<char>(kGemmWs);
  ML_TRY((pkm_topk_bwd_workspace(&s.pkm, &b.pkm_bytes)));
  b.pkm_ws = c.take<char>(b.pkm_bytes);
  b.dw_local = c.take<float>(int64_t(s.pkm.T) * s.pkm.H * s.pkm.k);
  return ML_OK;
}

mlStatus memory_layer_bwd_group_workspace(mlGroup g, const mlLayerShape* shape, size_t* bytes) {
  ML_API_BEGIN_X
  ML_TRY(check_layer_group(g, shape, ML_OUT_ALLTOALL));
  if (!bytes) return fail(ML_ERR_ARG, "null bytes");
  Carver c(nullptr);
  LayerBwdGroupBufs b;
  ML_TRY(layer_bwd_group_carve(c, g, *shape, b));
  *bytes = c.used;
  return ML_OK;
  ML_API_END_X
}

mlStatus memory_layer_bwd_group(mlGroup g, const mlLayerShape* shape, const void* dout,
                                const void* x, const void* q, const void* K1, const void* K2,
                                const void* V_shard, const void* W1, const void* W2,
                                const int32_t* idx_saved, const float* w_saved,
                                const int32_t* idx_all, const float* w_all, const void* g_saved,
                                const void* y_saved, const void* state, size_t state_bytes, void* dx,
                                float* dq, float* dK1, float* dK2, int32_t* dV_rows, void* dV_shard,
                                int32_t* U, float* dW1, float* dW2, float* dw_out, void* ws,
                                size_t ws_bytes, void* stream) {
  ML_API_BEGIN_X
  ML_TRY(check_layer_group(g, shape, ML_OUT_ALLTOALL));
  const mlLayerShape& s = *shape;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int T = s.pkm.T;
  if (!U) return fail(ML_ERR_ARG, "null U");
  if (T == 0) {
    ML_CUDA_TRY(cudaMemsetAsync(U, 0, sizeof(int32_t), st));
    return ML_OK;
  }
  if (!dout || !x || !q || !K1 || !K2 || !V_shard || !W1 || !W2 || !idx_saved || !w_saved ||
      !idx_all || !w_all || !g_saved || !y_saved || !dx || !dq || !dK1 || !dK2 || !dV_rows ||
      !dV_shard || !dW1 || !dW2 || !ws)
    return fail(ML_ERR_ARG, "null pointer argument");
  size_t need = 0;
  ML_TRY(memory_layer_bwd_group_workspace(g, shape, &need));
  if (ws_bytes < need) return fail(ML_ERR_WORKSPACE, "memory_layer_bwd_group: workspace too small");
  Carver c(ws);
  LayerBwdGroupBufs b;
  ML_TRY(layer_bwd_group_carve(c, g, s, b));
  const mlDtype dt = s.pkm.dtype;
  // gate backward (Eq. 2) on own tokens; weight gradients on the aux stream
  ML_TRY((ml_gemm(0, 1, T, s.dv, s.D, dout, s.D, W2, s.D, b.dz, s.dv, dt, 0, b.gemm_ws,
                              kGemmWs, st)));
  ML_TRY((ml_gate_bwd(b.dz, g_saved, y_saved, b.z, b.dy, b.dg, int64_t(T) * s.dv, dt, st)));
  cudaStream_t as = serial_mode() ? st : g->aux;
  ML_TRY(dep(st, as, g->ev[5]));
  ML_TRY((ml_gemm(1, 0, s.dv, s.D, T, b.z, s.dv, dout, s.D, dW2, s.D, dt, 1, b.gemm_ws2,
                              kGemmWs, as)));
  ML_TRY((ml_gemm(1, 0, s.D, s.dv, T, x, s.D, b.dg, s.dv, dW1, s.dv, dt, 1, b.gemm_ws2,
                              kGemmWs, as)));
  ML_TRY((ml_gemm(0, 1, T, s.D, s.dv, b.dg, s.dv, W1, s.dv, dx, s.D, dt, 0, b.gemm_ws2,
                              kGemmWs, as)));
  // bag backward over the group: dy slices all-to-all, local sorted
  // reduction (dV stays here), reduce-scatter of the partial dw
  const mlBagShape bag = bag_of_layer(s);
  size_t bw = 0;
  ML_TRY(embbag_bwd_group_workspace(g, &bag, ML_OUT_ALLTOALL, &bw));
  // b.bag was carved first from ws by the same bwd_carve, so the bag-level
  // call re-carves exactly that region from its start (b.bag.dy_send)
  ML_TRY((embbag_bwd_group(g, &bag, V_shard, idx_all, w_all, b.dy, ML_OUT_ALLTOALL, state,
                                       state_bytes, dV_rows, dV_shard, U, b.dw_local, b.bag.dy_send,
                                       bw, st)));
  ML_TRY((pkm_topk_bwd(&s.pkm, q, K1, K2, idx_saved, w_saved, b.dw_local, dq, dK1, dK2,
                                   b.pkm_ws, b.pkm_bytes, st)));
  if (dw_out)
    ML_CUDA_TRY(cudaMemcpyAsync(dw_out, b.dw_local, sizeof(float) * size_t(T) * s.pkm.H * s.pkm.k,
                                cudaMemcpyDeviceToDevice, st));
  return dep(as, st, g->ev[6]);                    // join the weight gradients
  ML_API_END_X
}

}  // extern "C"
