// sldg_peer.cu -- peer-mapped halo layers (SLDG_DIST_PEER_HALO; DESIGN.md §7 "Peer-mapped halos").
//
// A sweep along the sharded layer dim reads source rows i - i* - 1 and i - i* (P:214-219), so
// its first and last layers need up to `pad` layers owned by the ring neighbours.  The NCCL path
// copies those layers into this rank's pad layers before the boundary layers are swept.  Here
// the pad layers are not memory of their own: with the CUDA virtual-memory API each coefficient
// array is one reserved address range in which
//   the local layers are backed by this rank's physical allocations, split per section (the fp64
//   planes, then the fp32 planes) into a low chunk (layers [0, pad)), a middle chunk and a high
//   chunk (layers [layers - pad, layers)), and
//   the left pad is a second mapping of the LEFT neighbour's high chunk, the right pad one of the
//   RIGHT neighbour's low chunk (the same buffer of the ping-pong pair, the same section).
// The sweep kernels are unchanged: their TMA boxes that fall in a pad read the neighbour's HBM
// directly (over NVLink for another GPU), so the transfer happens inside the sweep, tile by tile,
// with no exchange step, no NCCL kernel and no SM reserve.  With world == 1 (forced halo) the
// neighbour is this rank itself: the pads alias its own opposite boundary layers.
//
// Ordering across ranks (world > 1): a sharded sweep reads the neighbours' CURRENT source
// buffer, so each rank's previous sweep must be complete before it starts, and the neighbours
// must not overwrite that buffer (their next sweep writes it: ping-pong) before it ends.  Both
// are one NCCL send/recv fence with the two ring neighbours on the grid's stream, before and
// after the sweep (a fence completes only once the peer's stream has reached it).
//
// Physical chunks must be multiples of the allocation granularity at granularity-aligned
// offsets: pad * u and layers * u are multiples of it for both sections' per-layer bytes u, on
// every rank (peer_halo_check).  Cross-process mapping (world > 1) exports each chunk as a POSIX
// file descriptor and hands them to the two ring neighbours over an abstract-namespace unix socket
// (SCM_RIGHTS; the socket names go round in an NCCL all-gather) -- no ptrace rights needed.
// SLDG_DIST_PEER_VIA_FD runs the export / socket / import / map route in one process (world == 1,
// tested); the all-gather, the fences and NVLink reads need two GPUs (tests/test_gpu_multi.py,
// skipped on one-GPU boxes).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <poll.h>
#include <stddef.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "sldg_internal.h"

namespace sldg {

namespace {

#define SLDG_DRV(name) decltype(&::name) name = nullptr
struct Driver {
    SLDG_DRV(cuMemGetAllocationGranularity);
    SLDG_DRV(cuMemCreate);
    SLDG_DRV(cuMemRelease);
    SLDG_DRV(cuMemAddressReserve);
    SLDG_DRV(cuMemAddressFree);
    SLDG_DRV(cuMemMap);
    SLDG_DRV(cuMemUnmap);
    SLDG_DRV(cuMemSetAccess);
    SLDG_DRV(cuMemExportToShareableHandle);
    SLDG_DRV(cuMemImportFromShareableHandle);
    bool ok = false;
};
#undef SLDG_DRV

const Driver& drv()
{
    static Driver d = [] {
        Driver r;
        bool ok = true;
        auto get = [&](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess || !*fn)
                ok = false;
        };
        get("cuMemGetAllocationGranularity", (void**)&r.cuMemGetAllocationGranularity);
        get("cuMemCreate", (void**)&r.cuMemCreate);
        get("cuMemRelease", (void**)&r.cuMemRelease);
        get("cuMemAddressReserve", (void**)&r.cuMemAddressReserve);
        get("cuMemAddressFree", (void**)&r.cuMemAddressFree);
        get("cuMemMap", (void**)&r.cuMemMap);
        get("cuMemUnmap", (void**)&r.cuMemUnmap);
        get("cuMemSetAccess", (void**)&r.cuMemSetAccess);
        get("cuMemExportToShareableHandle", (void**)&r.cuMemExportToShareableHandle);
        get("cuMemImportFromShareableHandle", (void**)&r.cuMemImportFromShareableHandle);
        r.ok = ok;
        return r;
    }();
    return d;
}

CUmemAllocationProp alloc_prop(int device, bool shareable)
{
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    p.requestedHandleTypes = shareable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
    return p;
}

// per-layer bytes of the two sections of one array (sldg_internal.h layout); u32 may be 0
void section_units(const Layout& L, size_t* u64, size_t* u32)
{
    *u64 = (size_t)L.L * 8 * (size_t)L.nd;
    *u32 = (size_t)L.L * 4 * (size_t)(L.K - L.nd);
}


// ---- descriptor passing over abstract unix sockets (SCM_RIGHTS) ------------------------------
constexpr int kFdSlots = 8;  // [b][s][low / high] edge chunks of one rank

std::string sock_name(long long pid, long long seq) { return "sldg-peer-" + std::to_string(pid) + "-" + std::to_string(seq); }

socklen_t sock_addr(const std::string& name, sockaddr_un* a)
{
    memset(a, 0, sizeof(*a));
    a->sun_family = AF_UNIX;
    memcpy(a->sun_path + 1, name.data(), name.size());  // sun_path[0] = 0: abstract namespace
    return (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + name.size());
}

bool send_fds(int sock, const int* fds)
{
    char present[kFdSlots];
    int valid[kFdSlots], nv = 0;
    for (int i = 0; i < kFdSlots; ++i) {
        present[i] = fds[i] >= 0;
        if (fds[i] >= 0) valid[nv++] = fds[i];
    }
    iovec iov = {present, sizeof(present)};
    msghdr msg = {};
    msg.msg_iov = &iov;
    msg.msg_iovlen = 1;
    alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int) * kFdSlots)] = {};
    if (nv) {
        msg.msg_control = cbuf;
        msg.msg_controllen = CMSG_SPACE(sizeof(int) * nv);
        cmsghdr* c = CMSG_FIRSTHDR(&msg);
        c->cmsg_level = SOL_SOCKET;
        c->cmsg_type = SCM_RIGHTS;
        c->cmsg_len = CMSG_LEN(sizeof(int) * nv);
        memcpy(CMSG_DATA(c), valid, sizeof(int) * nv);
    }
    return sendmsg(sock, &msg, MSG_NOSIGNAL) == (ssize_t)sizeof(present);
}

bool recv_fds(int sock, int* fds)
{
    char present[kFdSlots];
    iovec iov = {present, sizeof(present)};
    msghdr msg = {};
    msg.msg_iov = &iov;
    msg.msg_iovlen = 1;
    alignas(cmsghdr) char cbuf[CMSG_SPACE(sizeof(int) * kFdSlots)] = {};
    msg.msg_control = cbuf;
    msg.msg_controllen = sizeof(cbuf);
    for (int i = 0; i < kFdSlots; ++i) fds[i] = -1;
    if (recvmsg(sock, &msg, MSG_CMSG_CLOEXEC) != (ssize_t)sizeof(present)) return false;
    int got[kFdSlots], ng = 0;
    for (cmsghdr* c = CMSG_FIRSTHDR(&msg); c; c = CMSG_NXTHDR(&msg, c))
        if (c->cmsg_level == SOL_SOCKET && c->cmsg_type == SCM_RIGHTS) {
            ng = (int)((c->cmsg_len - CMSG_LEN(0)) / sizeof(int));
            memcpy(got, CMSG_DATA(c), sizeof(int) * ng);
        }
    for (int i = 0, j = 0; i < kFdSlots; ++i)
        if (present[i]) fds[i] = (j < ng) ? got[j++] : -1;
    return true;
}

// serves this rank's descriptors to the two neighbour connections (or stops when the listening
// socket is shut down, or after 60 s without a connection)
void serve_fds(int lsock, const int* fds)
{
    for (int served = 0; served < 2;) {
        pollfd p = {lsock, POLLIN, 0};
        if (poll(&p, 1, 60000) <= 0 || !(p.revents & POLLIN)) return;
        const int c = accept4(lsock, nullptr, nullptr, SOCK_CLOEXEC);
        if (c < 0) return;
        ucred cr = {};
        socklen_t crl = sizeof(cr);
        if (getsockopt(c, SOL_SOCKET, SO_PEERCRED, &cr, &crl) == 0 && cr.uid == getuid()) {  // same user only
            send_fds(c, fds);
            ++served;
        }
        close(c);
    }
}
}  // namespace

std::string peer_halo_check(const Layout& L, int world, size_t gran)
{
    if (L.D < 2) return "peer-mapped halos need D >= 2 (a sharded layer dim)";
    if (L.pad < 1) return "peer-mapped halos need pad >= 1";
    size_t u[2];
    section_units(L, &u[0], &u[1]);
    const int64_t n = L.n[L.D - 1];
    for (int r = 0; r < world; ++r) {
        const int64_t layers = n / world + ((r < n % world) ? 1 : 0);
        if (layers < 2 * L.pad)
            return "rank " + std::to_string(r) + " holds " + std::to_string(layers) + " layers < 2 * pad = " +
                   std::to_string(2 * L.pad) + " (its low and high chunks would overlap)";
        for (int s = 0; s < 2; ++s) {
            if (!u[s]) continue;
            if (((size_t)L.pad * u[s]) % gran || ((size_t)layers * u[s]) % gran)
                return std::string(s ? "fp32" : "fp64") + " section: pad * " + std::to_string(u[s]) + " B and " +
                       std::to_string(layers) + " layers * " + std::to_string(u[s]) +
                       " B must be multiples of the allocation granularity " + std::to_string(gran) + " B";
        }
    }
    return "";
}

size_t peer_granularity(int device)
{
    const Driver& d = drv();
    if (!d.ok) return 0;
    CUmemAllocationProp p = alloc_prop(device, false);
    size_t g = 0;
    if (d.cuMemGetAllocationGranularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS) return 0;
    return g;
}

}  // namespace sldg

using namespace sldg;

// Chunk bookkeeping of one grid (sldg_grid_s::peer)
struct sldg_peer_s {
    struct Map {
        CUdeviceptr va;
        size_t bytes;
    };
    CUdeviceptr base[2] = {0, 0};
    size_t bytes = 0;
    std::vector<CUmemGenericAllocationHandle> handles;  // created or imported here: released at free
    std::vector<Map> maps;
    // this rank's low / high chunk handles per (buffer, section): [b][s][0 = low, 1 = high]
    CUmemGenericAllocationHandle edge[2][2][2] = {};
    int* d_fence = nullptr;  // fence words (world > 1)
};

namespace sldg {

void peer_free(sldg_grid g)
{
    sldg_peer_s* P = g->peer;
    if (!P) return;
    const Driver& d = drv();
    for (const auto& m : P->maps) d.cuMemUnmap(m.va, m.bytes);
    for (auto h : P->handles) d.cuMemRelease(h);
    for (int b = 0; b < 2; ++b)
        if (P->base[b]) d.cuMemAddressFree(P->base[b], P->bytes);
    if (P->d_fence) cudaFree(P->d_fence);
    delete P;
    g->peer = nullptr;
    g->alloc[0] = g->alloc[1] = nullptr;
}

// Reserve both arrays, back their local layers with this rank's chunks, map the neighbours'
// edge chunks into the pads.  Returns "" or the reason (the caller destroys the grid).  With
// world > 1 this is collective: a rank that fails locally still takes part in the all-gather
// and the closing all-reduce (carrying its failure), so every rank returns the error together.
// via_fd (world == 1, testing): the rank's own chunks go through the descriptor export /
// unix-socket / import path of world > 1.
std::string peer_alloc(sldg_grid g, bool via_fd)
{
    const Layout& L = g->lay;
    const Driver& d = drv();
    if (!d.ok) return "the CUDA virtual-memory driver entry points are unavailable";
    const size_t gran = peer_granularity(g->device);
    if (!gran) return "cuMemGetAllocationGranularity failed";
    std::string why = peer_halo_check(L, g->world, gran);  // identical on every rank
    if (!why.empty()) return why;
    const bool multi = g->world > 1;
    const bool shared = multi || via_fd;
    CUmemAllocationProp prop = alloc_prop(g->device, shared);
    sldg_peer_s* P = new sldg_peer_s();
    g->peer = P;
    size_t u[2];
    section_units(L, &u[0], &u[1]);
    const size_t p = (size_t)L.pad, nl = (size_t)L.layers;
    const size_t sec_bytes[2] = {(nl + 2 * p) * u[0], (nl + 2 * p) * u[1]};
    P->bytes = sec_bytes[0] + sec_bytes[1];
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = g->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    auto map = [&](CUdeviceptr va, size_t bytes, CUmemGenericAllocationHandle h) -> bool {
        if (d.cuMemMap(va, bytes, 0, h, 0) != CUDA_SUCCESS) return false;
        P->maps.push_back({va, bytes});
        return d.cuMemSetAccess(va, bytes, &acc, 1) == CUDA_SUCCESS;
    };
    auto create = [&](size_t bytes, CUmemGenericAllocationHandle* h) -> bool {
        if (d.cuMemCreate(h, bytes, &prop, 0) != CUDA_SUCCESS) return false;
        P->handles.push_back(*h);
        return true;
    };
    // 1. local chunks
    std::string err;
    for (int b = 0; b < 2 && err.empty(); ++b) {
        if (d.cuMemAddressReserve(&P->base[b], P->bytes, gran, 0, 0) != CUDA_SUCCESS) {
            P->base[b] = 0;
            err = "cuMemAddressReserve of " + std::to_string(P->bytes) + " bytes failed";
            break;
        }
        size_t off = 0;
        for (int s = 0; s < 2 && err.empty(); ++s) {
            if (!u[s]) continue;
            const CUdeviceptr sec = P->base[b] + off;
            CUmemGenericAllocationHandle lo = 0, mid = 0, hi = 0;
            if (!create(p * u[s], &lo) || !map(sec + p * u[s], p * u[s], lo)) err = "low chunk allocation failed";
            else if (nl > 2 * p &&
                     (!create((nl - 2 * p) * u[s], &mid) || !map(sec + 2 * p * u[s], (nl - 2 * p) * u[s], mid)))
                err = "middle chunk allocation failed";
            else if (!create(p * u[s], &hi) || !map(sec + nl * u[s], p * u[s], hi)) err = "high chunk allocation failed";
            else if (cudaMemsetAsync((void*)(sec + p * u[s]), 0, nl * u[s], g->stream) != cudaSuccess)
                err = "memset failed";
            P->edge[b][s][0] = lo;
            P->edge[b][s][1] = hi;
            off += sec_bytes[s];
        }
    }
    if (err.empty() && cudaStreamSynchronize(g->stream) != cudaSuccess) err = "memset failed";
    if (!multi && !err.empty()) return err;
    // 2. the neighbours' edge chunks: nb[b][s][0] = left neighbour's high, [1] = right neighbour's low
    CUmemGenericAllocationHandle nb[2][2][2] = {};
    if (!shared) {
        for (int b = 0; b < 2; ++b)
            for (int s = 0; s < 2; ++s) {
                nb[b][s][0] = P->edge[b][s][1];
                nb[b][s][1] = P->edge[b][s][0];
            }
    } else {
        // export my 8 edge chunks as descriptors, listen on an abstract socket, all-gather its
        // name (pid, sequence number; pid -1 marks a failed rank), then fetch the neighbours'
        // descriptors from their sockets while a thread serves mine
        constexpr int kW = 2;
        static std::atomic<long long> seq_ctr{0};
        const long long seq = seq_ctr++;
        int my_fds[kFdSlots];
        for (int i = 0; i < kFdSlots; ++i) my_fds[i] = -1;
        int lsock = -1;
        if (err.empty()) {
            for (int b = 0; b < 2; ++b)
                for (int s = 0; s < 2; ++s)
                    for (int e = 0; e < 2 && err.empty(); ++e) {
                        if (!u[s]) continue;
                        int fd = -1;
                        if (d.cuMemExportToShareableHandle(&fd, P->edge[b][s][e],
                                                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS)
                            err = "cuMemExportToShareableHandle failed";
                        else
                            my_fds[(b * 2 + s) * 2 + e] = fd;
                    }
        }
        if (err.empty()) {
            sockaddr_un a;
            const socklen_t len = sock_addr(sock_name(getpid(), seq), &a);
            lsock = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
            if (lsock < 0 || bind(lsock, (sockaddr*)&a, len) != 0 || listen(lsock, 4) != 0)
                err = "cannot listen on the descriptor-exchange socket";
        }
        std::thread server;
        if (err.empty()) server = std::thread(serve_fds, lsock, my_fds);
        std::vector<long long> mine = {err.empty() ? (long long)getpid() : -1, seq};
        std::vector<long long> all((size_t)kW * g->world, -1);
        long long* dbuf = nullptr;
        bool comm_ok = true;
        if (multi) {
            ncclComm_t comm = (ncclComm_t)g->comm;
            comm_ok = cudaMalloc(&dbuf, sizeof(long long) * kW * (g->world + 1)) == cudaSuccess &&
                      cudaMemcpy(dbuf, mine.data(), sizeof(long long) * kW, cudaMemcpyHostToDevice) == cudaSuccess &&
                      ncclAllGather(dbuf, dbuf + kW, kW, ncclInt64, comm, g->stream) == ncclSuccess &&
                      cudaMemcpyAsync(all.data(), dbuf + kW, sizeof(long long) * kW * g->world,
                                      cudaMemcpyDeviceToHost, g->stream) == cudaSuccess &&
                      cudaStreamSynchronize(g->stream) == cudaSuccess;
        } else {
            all = mine;
        }
        bool any_failed = !comm_ok;
        for (int r = 0; r < g->world && comm_ok; ++r) any_failed |= all[(size_t)r * kW] < 0;
        const int left = (g->rank + g->world - 1) % g->world, right = (g->rank + 1) % g->world;
        std::vector<int> fetched;
        auto fetch = [&](int peer, int* fds) -> bool {  // the peer's 8 descriptors
            sockaddr_un a;
            const socklen_t len = sock_addr(sock_name(all[(size_t)peer * kW], all[(size_t)peer * kW + 1]), &a);
            const int c = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
            if (c < 0) return false;
            // the listener must be the process the all-gather named (SO_PEERCRED), not a squatter
            ucred cr = {};
            socklen_t crl = sizeof(cr);
            const bool ok = connect(c, (sockaddr*)&a, len) == 0 &&
                            getsockopt(c, SOL_SOCKET, SO_PEERCRED, &cr, &crl) == 0 &&
                            (long long)cr.pid == all[(size_t)peer * kW] && cr.uid == getuid() && recv_fds(c, fds);
            close(c);
            for (int i = 0; i < kFdSlots; ++i)
                if (fds[i] >= 0) fetched.push_back(fds[i]);
            return ok;
        };
        auto import = [&](int fd, CUmemGenericAllocationHandle* h) -> bool {
            if (fd < 0 || d.cuMemImportFromShareableHandle(h, (void*)(uintptr_t)fd,
                                                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) != CUDA_SUCCESS)
                return false;
            P->handles.push_back(*h);
            return true;
        };
        bool ok = !any_failed && err.empty();
        int lf[kFdSlots], rf[kFdSlots];
        if (ok) ok = fetch(left, lf) && fetch(right, rf);
        for (int b = 0; b < 2 && ok; ++b)
            for (int s = 0; s < 2 && ok; ++s) {
                if (!u[s]) continue;
                ok = import(lf[(b * 2 + s) * 2 + 1], &nb[b][s][0]) && import(rf[(b * 2 + s) * 2 + 0], &nb[b][s][1]);
            }
        if (err.empty() && !ok)
            err = any_failed ? "another rank failed to set up its peer-mapped halo chunks"
                             : "fetching or importing a neighbour's chunk failed (unix socket / cuMemImportFromShareableHandle)";
        // the sum of failures decides for all; a server whose neighbours gave up stops here
        if (multi && comm_ok) {
            int* flag = (int*)dbuf;
            const int mine_bad = err.empty() ? 0 : 1;
            int bad = 1;
            comm_ok = cudaMemcpy(flag, &mine_bad, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
                      ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, (ncclComm_t)g->comm, g->stream) == ncclSuccess &&
                      cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, g->stream) == cudaSuccess &&
                      cudaStreamSynchronize(g->stream) == cudaSuccess;
            if (err.empty() && (!comm_ok || bad)) err = "another rank failed to map its peer-mapped halo chunks";
        }
        if (multi && !comm_ok && err.empty()) err = "the chunk descriptor exchange failed";
        if (lsock >= 0) shutdown(lsock, SHUT_RDWR);  // wakes a server still waiting (failure paths)
        if (server.joinable()) server.join();
        if (lsock >= 0) close(lsock);
        for (int fd : fetched) close(fd);
        for (int i = 0; i < kFdSlots; ++i)
            if (my_fds[i] >= 0) close(my_fds[i]);
        if (dbuf) cudaFree(dbuf);
        if (!err.empty()) return err;
        if (multi) {
            if (cudaMalloc(&P->d_fence, 4 * sizeof(int)) != cudaSuccess) return "allocation failed";
            if (cudaMemset(P->d_fence, 0, 4 * sizeof(int)) != cudaSuccess) return "memset failed";
        }
    }
    // 3. the pads.  (world > 1: a failure here is local to a rank that already passed the
    // collective steps; its creation fails, the neighbours' grids stay valid)
    for (int b = 0; b < 2; ++b) {
        size_t off = 0;
        for (int s = 0; s < 2; ++s) {
            if (!u[s]) continue;
            const CUdeviceptr sec = P->base[b] + off;
            if (!map(sec, p * u[s], nb[b][s][0]) || !map(sec + (nl + p) * u[s], p * u[s], nb[b][s][1]))
                return "mapping a neighbour's edge chunk into the pad layers failed";
            off += sec_bytes[s];
        }
        g->alloc[b] = (void*)P->base[b];
    }
    return "";
}

// world > 1: one send/recv of a word with both ring neighbours on the grid's stream
cudaError_t peer_fence(sldg_grid g)
{
    if (g->world <= 1 || !g->peer) return cudaSuccess;
    ncclComm_t comm = (ncclComm_t)g->comm;
    const int left = (g->rank + g->world - 1) % g->world, right = (g->rank + 1) % g->world;
    int* f = g->peer->d_fence;
    bool ok = ncclGroupStart() == ncclSuccess && ncclSend(f, 1, ncclInt32, left, comm, g->stream) == ncclSuccess &&
              ncclSend(f + 1, 1, ncclInt32, right, comm, g->stream) == ncclSuccess &&
              ncclRecv(f + 2, 1, ncclInt32, left, comm, g->stream) == ncclSuccess &&
              ncclRecv(f + 3, 1, ncclInt32, right, comm, g->stream) == ncclSuccess && ncclGroupEnd() == ncclSuccess;
    return ok ? cudaSuccess : cudaErrorUnknown;
}

}  // namespace sldg
