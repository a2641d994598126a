// NCCL for the sharded applies (SURVEY.md §8(b) multi-GPU row), loaded at run time:
// libfdp does not link NCCL, so it loads (and its single-GPU entry points work) on a host without
// it; the first communicator dlopens libnccl.so.2 -- in a process that imported torch that is the
// copy torch already loaded (the loader matches the soname). Every NCCL failure is reported as
// FDP_ERR_NCCL with NCCL's own message.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "abi_impl.h"

namespace fdp {
namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi* api(std::string* why) {
  static NcclApi a;
  static bool ok = false;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      const char* e = dlerror();
      err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      if (!fn) {
        all = false;
        err = std::string("libnccl.so.2 lacks ") + name;
      }
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GetErrorString, "ncclGetErrorString");
    ok = all;
  });
  if (!ok) {
    if (why) *why = err;
    return nullptr;
  }
  return &a;
}

fdp_status nccl_fail(const NcclApi* a, ncclResult_t r, const char* where) {
  return fail(FDP_ERR_NCCL, std::string(where) + ": " + (a ? a->GetErrorString(r) : "NCCL unavailable"));
}

}  // namespace

static_assert(sizeof(ncclUniqueId) == FDP_NCCL_ID_BYTES, "ncclUniqueId size");

fdp_status nccl_unique_id(void* id) {
  std::string why;
  const NcclApi* a = api(&why);
  if (!a) return fail(FDP_ERR_NCCL, "fdp_nccl_unique_id: " + why);
  ncclUniqueId u;
  ncclResult_t r = a->GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(a, r, "fdp_nccl_unique_id");
  std::memcpy(id, &u, sizeof(u));
  return FDP_OK;
}

fdp_status nccl_comm_init(void** comm, int nranks, int rank, const void* id) {
  std::string why;
  const NcclApi* a = api(&why);
  if (!a) return fail(FDP_ERR_NCCL, "fdp_comm_init: " + why);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  ncclResult_t r = a->CommInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) return nccl_fail(a, r, "fdp_comm_init: ncclCommInitRank");
  *comm = c;
  return FDP_OK;
}

void nccl_comm_destroy(void* comm) {
  const NcclApi* a = api(nullptr);
  if (a && comm) a->CommDestroy(static_cast<ncclComm_t>(comm));
}

fdp_status nccl_exchange(void* comm, const std::vector<NcclXfer>& xs, cudaStream_t s, const char* where) {
  const NcclApi* a = api(nullptr);
  if (!a || !comm) return fail(FDP_ERR_NCCL, std::string(where) + ": no NCCL communicator");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = a->GroupStart();
  if (r != ncclSuccess) return nccl_fail(a, r, where);
  for (const NcclXfer& x : xs) {
    if (x.count == 0) continue;
    r = x.send ? a->Send(x.buf, (size_t)x.count, ncclDouble, x.peer, c, s)
               : a->Recv(const_cast<double*>(x.buf), (size_t)x.count, ncclDouble, x.peer, c, s);
    if (r != ncclSuccess) {
      a->GroupEnd();
      return nccl_fail(a, r, where);
    }
  }
  r = a->GroupEnd();
  if (r != ncclSuccess) return nccl_fail(a, r, where);
  return FDP_OK;
}

}  // namespace fdp
