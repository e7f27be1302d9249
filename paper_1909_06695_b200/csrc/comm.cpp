// Distributed context, point-to-point transfers and state export/import of
// the C ABI (rp_ctx_create(device, nccl_unique_id, rank, nranks),
// rp_send / rp_recv on a caller stream, rp_export_state / rp_import_state).
//
// The reference runs its modules as threads of one process and hands
// activations / boundary gradients over by reference (engine.py:246-265,
// 313-373); across GPUs the same hand-offs are NCCL point-to-point transfers
// over NVLink.  NCCL is resolved at run time (dlopen of RP_NCCL_LIB, else
// libnccl.so.2 -- torch's bundled copy when the host already loaded it), so
// the library links no communication runtime and a single-GPU host never
// needs one.
//
// State export/import writes and reads the RPCK container of the reference's
// checkpoint.py:1-70 (runner.py:111-226 names the entries): a C host can
// checkpoint the rings, slots, boundary gradients and moments it owns and a
// Python host (or the reference) can read them back, and vice versa.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "rp_internal.h"

namespace {

// ---- NCCL, resolved at run time --------------------------------------------
struct NcclId {
  char internal[128];
};
typedef void* NcclComm;
typedef int NcclResult;
struct Nccl {
  NcclResult (*get_unique_id)(NcclId*) = nullptr;
  NcclResult (*comm_init_rank)(NcclComm*, int, NcclId, int) = nullptr;
  NcclResult (*comm_destroy)(NcclComm) = nullptr;
  NcclResult (*send)(const void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  NcclResult (*recv)(void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  NcclResult (*group_start)() = nullptr;
  NcclResult (*group_end)() = nullptr;
  const char* (*error_string)(NcclResult) = nullptr;
  bool ok = false;
  std::string why;
};
constexpr int kNcclInt8 = 0;  // ncclInt8: byte transfers

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("RP_NCCL_LIB");
    void* h = nullptr;
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (!name) continue;
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      n.why = "NCCL library not found (set RP_NCCL_LIB)";
      return;
    }
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.send = reinterpret_cast<decltype(n.send)>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(h, "ncclRecv"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(h, "ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.send && n.recv && n.group_start &&
           n.group_end && n.error_string;
    if (!n.ok) n.why = "NCCL library lacks the point-to-point API";
  });
  return n;
}

int nccl_check(NcclResult r, const char* what) {
  if (r == 0) return RP_OK;
  return rp::set_error(RP_ERR_NCCL, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "NCCL error");
}

}  // namespace

struct rp_ctx {
  int device, rank, nranks;
  NcclComm comm;
};

extern "C" {

int rp_nccl_unique_id(void* id128) {
  Nccl& n = nccl();
  if (!n.ok) return rp::set_error(RP_ERR_NCCL, "%s", n.why.c_str());
  if (!id128) return rp::set_error(RP_ERR_INVALID, "rp_nccl_unique_id: null buffer");
  NcclId id;
  if (int e = nccl_check(n.get_unique_id(&id), "ncclGetUniqueId")) return e;
  std::memcpy(id128, &id, sizeof(id));
  return RP_OK;
}

int rp_ctx_create(int32_t device, const void* nccl_unique_id, int32_t rank, int32_t nranks, rp_ctx** out) {
  if (!out || !nccl_unique_id) return rp::set_error(RP_ERR_INVALID, "rp_ctx_create: null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return rp::set_error(RP_ERR_INVALID, "rp_ctx_create: rank %d of %d", rank, nranks);
  Nccl& n = nccl();
  if (!n.ok) return rp::set_error(RP_ERR_NCCL, "%s", n.why.c_str());
  if (cudaSetDevice(device) != cudaSuccess) return rp::set_error(RP_ERR_CUDA, "rp_ctx_create: device %d", device);
  NcclId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  NcclComm comm = nullptr;
  if (int e = nccl_check(n.comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank")) return e;
  *out = new rp_ctx{device, rank, nranks, comm};
  return RP_OK;
}

int rp_ctx_destroy(rp_ctx* ctx) {
  if (!ctx) return RP_OK;
  int e = RP_OK;
  if (ctx->comm) e = nccl_check(nccl().comm_destroy(ctx->comm), "ncclCommDestroy");
  delete ctx;
  return e;
}

int rp_ctx_rank(const rp_ctx* ctx) { return ctx ? ctx->rank : -1; }
int rp_ctx_nranks(const rp_ctx* ctx) { return ctx ? ctx->nranks : -1; }

int rp_send(rp_ctx* ctx, const void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!ctx || (!buf && bytes)) return rp::set_error(RP_ERR_INVALID, "rp_send: null argument");
  if (peer < 0 || peer >= ctx->nranks) return rp::set_error(RP_ERR_INVALID, "rp_send: peer %d", peer);
  return nccl_check(nccl().send(buf, (size_t)bytes, kNcclInt8, peer, ctx->comm, static_cast<cudaStream_t>(stream)),
                    "ncclSend");
}

int rp_recv(rp_ctx* ctx, void* buf, int64_t bytes, int32_t peer, void* stream) {
  if (!ctx || (!buf && bytes)) return rp::set_error(RP_ERR_INVALID, "rp_recv: null argument");
  if (peer < 0 || peer >= ctx->nranks) return rp::set_error(RP_ERR_INVALID, "rp_recv: peer %d", peer);
  return nccl_check(nccl().recv(buf, (size_t)bytes, kNcclInt8, peer, ctx->comm, static_cast<cudaStream_t>(stream)),
                    "ncclRecv");
}

int rp_group_start(void) {
  Nccl& n = nccl();
  if (!n.ok) return rp::set_error(RP_ERR_NCCL, "%s", n.why.c_str());
  return nccl_check(n.group_start(), "ncclGroupStart");
}

int rp_group_end(void) {
  Nccl& n = nccl();
  if (!n.ok) return rp::set_error(RP_ERR_NCCL, "%s", n.why.c_str());
  return nccl_check(n.group_end(), "ncclGroupEnd");
}

}  // extern "C"

// ---- state export / import (RPCK container) ---------------------------------
namespace {

constexpr char kMagic[4] = {'R', 'P', 'C', 'K'};
constexpr uint32_t kVersion = 1;

int esize_of(int32_t dt) {
  switch (dt) {
    case RP_F32: return 4;
    case RP_BF16: return 2;
    case RP_I64: return 8;
    case RP_U64: return 8;
    case RP_F64: return 8;
    default: return 0;
  }
}
int tag_of(int32_t dt) { return (dt == RP_I64) ? 1 : (dt == RP_U64 ? 2 : 0); }  // f8 / i8 / u8

int64_t numel(const rp_state_entry& e) {
  int64_t n = 1;
  for (int i = 0; i < e.ndim; ++i) n *= e.shape[i];
  return n;
}

int check_entry(const rp_state_entry& e) {
  if (!e.name || !*e.name) return rp::set_error(RP_ERR_INVALID, "state entry without a name");
  if (e.ndim < 0 || e.ndim > 4) return rp::set_error(RP_ERR_INVALID, "state entry %s: ndim %d", e.name, e.ndim);
  if (!esize_of(e.dtype)) return rp::set_error(RP_ERR_INVALID, "state entry %s: dtype %d", e.name, e.dtype);
  if (numel(e) && !e.ptr) return rp::set_error(RP_ERR_INVALID, "state entry %s: null pointer", e.name);
  return RP_OK;
}

int64_t entry_bytes(const rp_state_entry& e) {
  return 2 + (int64_t)std::strlen(e.name) + 2 + 8LL * e.ndim + 8 * numel(e);
}

int copy_raw(void* dst, const void* src, int64_t bytes, bool to_host, const rp_state_entry& e, cudaStream_t st) {
  if (!bytes) return RP_OK;
  if (e.on_host) {
    std::memcpy(dst, src, (size_t)bytes);
    return RP_OK;
  }
  if (cudaMemcpyAsync(dst, src, (size_t)bytes, to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return rp::set_error(RP_ERR_CUDA, "state entry %s: copy failed", e.name);
  return RP_OK;
}

float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
uint16_t f64_to_bf16(double x) {  // round to nearest even (NaN kept quiet)
  float f = (float)x;
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

}  // namespace

extern "C" {

int64_t rp_state_bytes(const rp_state_entry* entries, int32_t n) {
  int64_t b = 12;
  for (int i = 0; i < n; ++i) {
    if (check_entry(entries[i])) return -1;
    b += entry_bytes(entries[i]);
  }
  return b;
}

int rp_export_state(const rp_state_entry* entries, int32_t n, void* blob, int64_t blob_bytes, void* stream) {
  if (!entries && n) return rp::set_error(RP_ERR_INVALID, "rp_export_state: null entries");
  const int64_t need = rp_state_bytes(entries, n);
  if (need < 0) return RP_ERR_INVALID;
  if (!blob || blob_bytes < need)
    return rp::set_error(RP_ERR_INVALID, "rp_export_state: blob needs %lld bytes", (long long)need);
  char* p = static_cast<char*>(blob);
  std::memcpy(p, kMagic, 4);
  std::memcpy(p + 4, &kVersion, 4);
  const uint32_t cnt = (uint32_t)n;
  std::memcpy(p + 8, &cnt, 4);
  p += 12;
  std::vector<char> raw;
  for (int i = 0; i < n; ++i) {
    const rp_state_entry& e = entries[i];
    const uint16_t len = (uint16_t)std::strlen(e.name);
    std::memcpy(p, &len, 2);
    std::memcpy(p + 2, e.name, len);
    p += 2 + len;
    p[0] = (char)tag_of(e.dtype);
    p[1] = (char)e.ndim;
    p += 2;
    for (int k = 0; k < e.ndim; ++k) {
      std::memcpy(p, &e.shape[k], 8);
      p += 8;
    }
    const int64_t cnt_e = numel(e), es = esize_of(e.dtype);
    raw.resize((size_t)(cnt_e * es));
    if (int r = copy_raw(raw.data(), e.ptr, cnt_e * es, true, e, static_cast<cudaStream_t>(stream))) return r;
    // widen to the container's 8-byte types (exact for every dtype here)
    for (int64_t j = 0; j < cnt_e; ++j) {
      if (e.dtype == RP_F32) {
        float f;
        std::memcpy(&f, raw.data() + 4 * j, 4);
        const double v = f;
        std::memcpy(p + 8 * j, &v, 8);
      } else if (e.dtype == RP_BF16) {
        uint16_t h;
        std::memcpy(&h, raw.data() + 2 * j, 2);
        const double v = bf16_to_f32(h);
        std::memcpy(p + 8 * j, &v, 8);
      } else {
        std::memcpy(p + 8 * j, raw.data() + 8 * j, 8);
      }
    }
    p += 8 * cnt_e;
  }
  return RP_OK;
}

int rp_import_state(const rp_state_entry* entries, int32_t n, const void* blob, int64_t blob_bytes, void* stream) {
  const char* b = static_cast<const char*>(blob);
  if (!b || blob_bytes < 12 || std::memcmp(b, kMagic, 4) != 0)
    return rp::set_error(RP_ERR_INVALID, "rp_import_state: not an RPCK container");
  uint32_t ver, cnt;
  std::memcpy(&ver, b + 4, 4);
  std::memcpy(&cnt, b + 8, 4);
  if (ver != kVersion) return rp::set_error(RP_ERR_INVALID, "rp_import_state: container version %u", ver);
  // index the container
  struct Item {
    std::string name;
    int tag, ndim;
    int64_t shape[8];
    const char* data;
    int64_t count;
  };
  std::vector<Item> items;
  int64_t pos = 12;
  for (uint32_t i = 0; i < cnt; ++i) {
    Item it;
    if (pos + 2 > blob_bytes) return rp::set_error(RP_ERR_INVALID, "rp_import_state: truncated container");
    uint16_t len;
    std::memcpy(&len, b + pos, 2);
    pos += 2;
    if (pos + len + 2 > blob_bytes) return rp::set_error(RP_ERR_INVALID, "rp_import_state: truncated container");
    it.name.assign(b + pos, len);
    pos += len;
    it.tag = (unsigned char)b[pos];
    it.ndim = (unsigned char)b[pos + 1];
    pos += 2;
    if (it.ndim > 8 || pos + 8LL * it.ndim > blob_bytes)
      return rp::set_error(RP_ERR_INVALID, "rp_import_state: bad entry %s", it.name.c_str());
    it.count = 1;
    for (int k = 0; k < it.ndim; ++k) {
      std::memcpy(&it.shape[k], b + pos, 8);
      it.count *= it.shape[k];
      pos += 8;
    }
    it.data = b + pos;
    pos += 8 * it.count;
    if (pos > blob_bytes) return rp::set_error(RP_ERR_INVALID, "rp_import_state: truncated entry %s", it.name.c_str());
    items.push_back(it);
  }
  std::vector<char> raw;
  for (int i = 0; i < n; ++i) {
    const rp_state_entry& e = entries[i];
    if (int r = check_entry(e)) return r;
    const Item* it = nullptr;
    for (const Item& c : items)
      if (c.name == e.name) it = &c;
    if (!it) return rp::set_error(RP_ERR_INVALID, "rp_import_state: container lacks %s", e.name);
    const int64_t cnt_e = numel(e), es = esize_of(e.dtype);
    if (it->count != cnt_e)
      return rp::set_error(RP_ERR_DIMENSION, "rp_import_state: %s has %lld elements, expected %lld", e.name,
                           (long long)it->count, (long long)cnt_e);
    if ((it->tag == 0) != (e.dtype == RP_F32 || e.dtype == RP_BF16 || e.dtype == RP_F64))
      return rp::set_error(RP_ERR_INVALID, "rp_import_state: %s dtype mismatch", e.name);
    raw.resize((size_t)(cnt_e * es));
    for (int64_t j = 0; j < cnt_e; ++j) {
      if (e.dtype == RP_F32 || e.dtype == RP_BF16) {
        double v;
        std::memcpy(&v, it->data + 8 * j, 8);
        if (e.dtype == RP_F32) {
          const float f = (float)v;
          std::memcpy(raw.data() + 4 * j, &f, 4);
        } else {
          const uint16_t h = f64_to_bf16(v);
          std::memcpy(raw.data() + 2 * j, &h, 2);
        }
      } else {
        std::memcpy(raw.data() + 8 * j, it->data + 8 * j, 8);
      }
    }
    if (int r = copy_raw(e.ptr, raw.data(), cnt_e * es, false, e, static_cast<cudaStream_t>(stream))) return r;
  }
  return RP_OK;
}

}  // extern "C"
