// cmn_nvls.cpp -- NEXT-3: NVLink SHARP (NVLS) multicast resources for the
// in-switch all-reduce (multimem.ld_reduce / multimem.st).
//
// One multicast object per communicator spans a per-rank physical allocation
// [packed (L x 4 B) | reduced (L x 4 B)].  Every rank maps its own allocation
// (unicast VA: the pack writes it, the update reads it) and the multicast
// object (multicast VA: the all-reduce kernel's ld_reduce / st).  Rank 0
// creates the object and hands its POSIX file descriptor to the other ranks
// over a Unix-domain socket (SCM_RIGHTS); the socket name travels through the
// caller's bootstrap allgather.  The CUDA driver API is reached through
// cudaGetDriverEntryPoint, so the library never links libcuda directly.
#include "cmn_nvls.h"

#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

namespace cmn {
namespace {

struct Drv {
    bool ok = false;
    CUresult (*MulticastCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *) = nullptr;
    CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
    CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle,
                                 size_t, size_t, unsigned long long) = nullptr;
    CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
    CUresult (*MulticastGetGranularity)(size_t *, const CUmulticastObjectProp *,
                                        CUmulticastGranularity_flags) = nullptr;
    CUresult (*MemCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *,
                          unsigned long long) = nullptr;
    CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*MemGetAllocationGranularity)(size_t *, const CUmemAllocationProp *,
                                            CUmemAllocationGranularity_flags) = nullptr;
    CUresult (*MemAddressReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
    CUresult (*MemExportToShareableHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                           unsigned long long) = nullptr;
    CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle *, void *,
                                             CUmemAllocationHandleType) = nullptr;
    CUresult (*DeviceGet)(CUdevice *, int) = nullptr;
    CUresult (*DeviceGetAttribute)(int *, CUdevice_attribute, CUdevice) = nullptr;
};

template <typename F>
bool sym(const char *name, F &f) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
    f = reinterpret_cast<F>(p);
    return true;
}

Drv &drv() {
    static Drv d;
    static bool tried = false;
    if (!tried) {
        tried = true;
        d.ok = sym("cuMulticastCreate", d.MulticastCreate) && sym("cuMulticastAddDevice", d.MulticastAddDevice) &&
               sym("cuMulticastBindMem", d.MulticastBindMem) && sym("cuMulticastUnbind", d.MulticastUnbind) &&
               sym("cuMulticastGetGranularity", d.MulticastGetGranularity) && sym("cuMemCreate", d.MemCreate) &&
               sym("cuMemRelease", d.MemRelease) &&
               sym("cuMemGetAllocationGranularity", d.MemGetAllocationGranularity) &&
               sym("cuMemAddressReserve", d.MemAddressReserve) && sym("cuMemAddressFree", d.MemAddressFree) &&
               sym("cuMemMap", d.MemMap) && sym("cuMemUnmap", d.MemUnmap) && sym("cuMemSetAccess", d.MemSetAccess) &&
               sym("cuMemExportToShareableHandle", d.MemExportToShareableHandle) &&
               sym("cuMemImportFromShareableHandle", d.MemImportFromShareableHandle) &&
               sym("cuDeviceGet", d.DeviceGet) && sym("cuDeviceGetAttribute", d.DeviceGetAttribute);
    }
    return d;
}

#define DRV(call, what)                                                            \
    do {                                                                           \
        CUresult r_ = (call);                                                      \
        if (r_ != CUDA_SUCCESS) {                                                  \
            err = std::string(what) + " failed (CUresult " + std::to_string(r_) + ")"; \
            return false;                                                          \
        }                                                                          \
    } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

// ------------------------------------------------------------- fd passing
// Rank 0 listens on an abstract Unix socket whose name it allgathers; every
// other rank connects and receives `fd` via SCM_RIGHTS.
bool share_fd(int rank, int world, cmn_allgather_fn ag, void *user, int fd_in, int *fd_out,
              std::string &err) {
    struct Name {
        int ok;           // rank 0 is listening (else every rank fails together)
        char path[92];
    };
    *fd_out = -1;
    if (world == 1) {
        *fd_out = fd_in;
        return true;
    }
    int lsock = -1;
    Name mine{};
    if (rank == 0) [&] {
        lsock = ::socket(AF_UNIX, SOCK_STREAM, 0);
        if (lsock < 0) {
            err = "socket() failed";
            return;
        }
        std::random_device rd;
        std::snprintf(mine.path, sizeof mine.path, "cmn-nvls-%d-%08x%08x", static_cast<int>(getpid()),
                      rd(), rd());
        sockaddr_un a{};
        a.sun_family = AF_UNIX;
        a.sun_path[0] = '\0';   // abstract namespace: nothing on the filesystem
        std::strncpy(a.sun_path + 1, mine.path, sizeof(a.sun_path) - 2);
        const socklen_t alen = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + std::strlen(mine.path));
        if (::bind(lsock, reinterpret_cast<sockaddr *>(&a), alen) != 0 || ::listen(lsock, world) != 0) {
            ::close(lsock);
            lsock = -1;
            err = "bind/listen on the abstract Unix socket failed";
            return;
        }
        mine.ok = 1;
    }();
    std::vector<Name> all(world);
    if (ag(&mine, all.data(), sizeof(Name), user) != 0) {
        if (lsock >= 0) ::close(lsock);
        err = "allgather callback failed";
        return false;
    }
    if (!all[0].ok) {
        if (rank != 0) err = "rank 0 could not open the fd hand-off socket";
        return false;
    }
    if (rank == 0) {
        for (int i = 1; i < world; ++i) {
            pollfd pf{lsock, POLLIN, 0};
            if (::poll(&pf, 1, 30000) != 1) {   // a peer that never connects must not hang us
                ::close(lsock);
                err = "timed out waiting for a peer to fetch the multicast fd";
                return false;
            }
            const int s = ::accept(lsock, nullptr, nullptr);
            if (s < 0) {
                ::close(lsock);
                err = "accept() failed";
                return false;
            }
            char byte = 'x';
            iovec io{&byte, 1};
            char ctrl[CMSG_SPACE(sizeof(int))] = {};
            msghdr m{};
            m.msg_iov = &io;
            m.msg_iovlen = 1;
            m.msg_control = ctrl;
            m.msg_controllen = sizeof ctrl;
            cmsghdr *cm = CMSG_FIRSTHDR(&m);
            cm->cmsg_level = SOL_SOCKET;
            cm->cmsg_type = SCM_RIGHTS;
            cm->cmsg_len = CMSG_LEN(sizeof(int));
            std::memcpy(CMSG_DATA(cm), &fd_in, sizeof(int));
            const ssize_t n = ::sendmsg(s, &m, 0);
            ::close(s);
            if (n != 1) {
                ::close(lsock);
                err = "sendmsg(SCM_RIGHTS) failed";
                return false;
            }
        }
        ::close(lsock);
        *fd_out = fd_in;
        return true;
    }
    const int s = ::socket(AF_UNIX, SOCK_STREAM, 0);
    if (s < 0) {
        err = "socket() failed";
        return false;
    }
    sockaddr_un a{};
    a.sun_family = AF_UNIX;
    std::strncpy(a.sun_path + 1, all[0].path, sizeof(a.sun_path) - 2);
    const socklen_t alen = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + std::strlen(all[0].path));
    bool connected = false;
    for (int attempt = 0; attempt < 3000 && !connected; ++attempt) {   // <= 30 s
        if (::connect(s, reinterpret_cast<sockaddr *>(&a), alen) == 0) {
            connected = true;
            break;
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
    if (!connected) {
        ::close(s);
        err = "connect() to rank 0's socket failed";
        return false;
    }
    char byte = 0;
    iovec io{&byte, 1};
    char ctrl[CMSG_SPACE(sizeof(int))] = {};
    msghdr m{};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof ctrl;
    const ssize_t n = ::recvmsg(s, &m, 0);
    ::close(s);
    cmsghdr *cm = CMSG_FIRSTHDR(&m);
    if (n != 1 || !cm || cm->cmsg_type != SCM_RIGHTS) {
        err = "recvmsg(SCM_RIGHTS) failed";
        return false;
    }
    std::memcpy(fd_out, CMSG_DATA(cm), sizeof(int));
    return true;
}

// ------------------------------------------------------------------ setup

bool nvls_supported(int device, std::string &err) {
    Drv &d = drv();
    if (!d.ok) {
        err = "driver multicast entry points unavailable";
        return false;
    }
    CUdevice dev;
    int v = 0;
    if (d.DeviceGet(&dev, device) != CUDA_SUCCESS ||
        d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS || !v) {
        err = "device does not support multicast (NVLS needs NVSwitch)";
        return false;
    }
    return true;
}

namespace {
// Every rank learns whether every rank succeeded so far, so a local failure
// never leaves the peers blocked in a later collective step (the fd
// hand-off, or cuMulticastBindMem, which waits for all devices to join).
bool agree(int world, cmn_allgather_fn ag, void *user, bool ok, std::string &err) {
    if (world == 1) return ok;
    // 1 = ok, 2 = multicast unsupported here, 0 = other failure; every rank
    // reports the same class (the caller maps "support" to UNSUPPORTED)
    std::vector<int> all(world);
    int mine = ok ? 1 : (err.find("support") != std::string::npos ? 2 : 0);
    if (ag(&mine, all.data(), sizeof(int), user) != 0) {
        err = "allgather callback failed";
        return false;
    }
    int worst = 1;
    for (int v : all)
        if (v != 1 && (worst == 1 || v == 2)) worst = v;
    if (worst == 1) return true;
    if (ok) err = worst == 2 ? "multicast not supported on another rank" : "NVLS setup failed on another rank";
    return false;
}
}  // namespace

bool nvls_setup(Nvls &n, int rank, int world, int device, size_t bytes_per_buffer,
                cmn_allgather_fn ag, void *user, std::string &err) {
    Drv &d = drv();
    CUdevice dev = 0;
    CUmulticastObjectProp mp{};
    CUmemAllocationProp ap{};
    size_t gran = 0;
    int fd = -1, fd_local = -1;
    // Stage 1: capability, sizes; rank 0 creates and exports the multicast object.
    const bool ok1 = [&]() -> bool {
        if (!nvls_supported(device, err)) return false;
        DRV(d.DeviceGet(&dev, device), "cuDeviceGet");
        mp.numDevices = static_cast<unsigned>(world);
        mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        mp.size = 2 * bytes_per_buffer;
        size_t g_mc = 0, g_mem = 0;
        DRV(d.MulticastGetGranularity(&g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED),
            "cuMulticastGetGranularity");
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = device;
        ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        DRV(d.MemGetAllocationGranularity(&g_mem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
            "cuMemGetAllocationGranularity");
        gran = g_mc > g_mem ? g_mc : g_mem;
        n.buffer_bytes = align_up(bytes_per_buffer, gran);
        n.size = 2 * n.buffer_bytes;
        mp.size = n.size;
        if (rank != 0) return true;
        const CUresult rc = d.MulticastCreate(&n.mc, &mp);
        if (rc != CUDA_SUCCESS) {
            // Observed on single-GPU boxes whose NVSwitch fabric is not set up
            // (nvidia-smi: GPU Fabric GUID 0): the attribute says "supported"
            // but every property combination is refused.
            err = "multicast object creation not supported here (cuMulticastCreate CUresult " +
                  std::to_string(rc) + "; NVSwitch fabric unavailable?)";
            return false;
        }
        n.have_mc = true;
        if (world > 1)
            DRV(d.MemExportToShareableHandle(&fd, n.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                "cuMemExportToShareableHandle");
        return true;
    }();
    if (!agree(world, ag, user, ok1, err)) {
        if (fd >= 0) ::close(fd);
        return false;
    }
    // Stage 2: hand the fd to the other ranks, import, join the team.
    bool ok2 = true;
    if (world > 1) {
        ok2 = share_fd(rank, world, ag, user, fd, &fd_local, err);
        if (rank == 0 && fd >= 0) ::close(fd);
    }
    ok2 = ok2 && [&]() -> bool {
        if (world > 1 && rank != 0) {
            const CUresult rc = d.MemImportFromShareableHandle(
                &n.mc, reinterpret_cast<void *>(static_cast<intptr_t>(fd_local)),
                CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
            ::close(fd_local);
            if (rc != CUDA_SUCCESS) {
                err = "cuMemImportFromShareableHandle failed (CUresult " + std::to_string(rc) + ")";
                return false;
            }
            n.have_mc = true;
        }
        DRV(d.MulticastAddDevice(n.mc, dev), "cuMulticastAddDevice");
        return true;
    }();
    if (!agree(world, ag, user, ok2, err)) return false;
    // Stage 3: bind this rank's memory (waits until every device joined), map
    // unicast and multicast views, zero the buffers.
    const bool ok3 = [&]() -> bool {
        DRV(d.MemCreate(&n.mem, n.size, &ap, 0), "cuMemCreate");
        n.have_mem = true;
        DRV(d.MulticastBindMem(n.mc, 0, n.mem, 0, n.size, 0), "cuMulticastBindMem");
        n.bound = true;
        n.device = device;
        CUmemAccessDesc acc{};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = device;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CUdeviceptr uc = 0, mc = 0;
        DRV(d.MemAddressReserve(&uc, n.size, gran, 0, 0), "cuMemAddressReserve(uc)");
        n.uc = reinterpret_cast<char *>(uc);
        DRV(d.MemMap(uc, n.size, 0, n.mem, 0), "cuMemMap(uc)");
        n.uc_mapped = true;
        DRV(d.MemSetAccess(uc, n.size, &acc, 1), "cuMemSetAccess(uc)");
        DRV(d.MemAddressReserve(&mc, n.size, gran, 0, 0), "cuMemAddressReserve(mc)");
        n.mcva = reinterpret_cast<char *>(mc);
        DRV(d.MemMap(mc, n.size, 0, n.mc, 0), "cuMemMap(mc)");
        n.mc_mapped = true;
        DRV(d.MemSetAccess(mc, n.size, &acc, 1), "cuMemSetAccess(mc)");
        if (cudaMemset(n.uc, 0, n.size) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
            err = "cudaMemset of the NVLS buffer failed";
            return false;
        }
        return true;
    }();
    return agree(world, ag, user, ok3, err);
}

void nvls_teardown(Nvls &n) {
    Drv &d = drv();
    if (!d.ok) return;
    cudaDeviceSynchronize();
    if (n.mc_mapped) d.MemUnmap(reinterpret_cast<CUdeviceptr>(n.mcva), n.size);
    if (n.mcva) d.MemAddressFree(reinterpret_cast<CUdeviceptr>(n.mcva), n.size);
    if (n.uc_mapped) d.MemUnmap(reinterpret_cast<CUdeviceptr>(n.uc), n.size);
    if (n.uc) d.MemAddressFree(reinterpret_cast<CUdeviceptr>(n.uc), n.size);
    if (n.bound) {
        CUdevice dev;
        if (d.DeviceGet(&dev, n.device) == CUDA_SUCCESS) d.MulticastUnbind(n.mc, dev, 0, n.size);
    }
    if (n.have_mem) d.MemRelease(n.mem);
    if (n.have_mc) d.MemRelease(n.mc);
    n = Nvls{};
}

}  // namespace cmn
