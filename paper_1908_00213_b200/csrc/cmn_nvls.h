// cmn_nvls.h -- NVLS (NVLink SHARP multicast) resources, host side.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/cmn.h"

namespace cmn {

struct Nvls {
    unsigned long long mc = 0;    // CUmemGenericAllocationHandle of the multicast object
    unsigned long long mem = 0;   // this rank's physical allocation bound to it
    bool have_mc = false, have_mem = false, bound = false, uc_mapped = false, mc_mapped = false;
    int device = 0;
    size_t size = 0;              // bytes mapped (2 buffers)
    size_t buffer_bytes = 0;      // bytes per buffer (packed | reduced), granularity-aligned
    char *uc = nullptr;           // unicast VA of this rank's allocation
    char *mcva = nullptr;         // multicast VA (ld_reduce / st address)
    bool ready() const { return mc_mapped; }
    void *packed_uc() const { return uc; }
    void *reduced_uc() const { return uc + buffer_bytes; }
    void *packed_mc() const { return mcva; }
    void *reduced_mc() const { return mcva + buffer_bytes; }
};

bool nvls_supported(int device, std::string &err);

// Collective across the communicator: rank 0 creates the multicast object and
// passes its POSIX fd to the other ranks (abstract Unix socket, SCM_RIGHTS;
// the socket name goes through `ag`), every rank adds its device, binds a
// 2 x bytes_per_buffer allocation and maps unicast + multicast VAs.
bool nvls_setup(Nvls &n, int rank, int world, int device, size_t bytes_per_buffer,
                cmn_allgather_fn ag, void *user, std::string &err);

void nvls_teardown(Nvls &n);

// File-descriptor hand-off used by nvls_setup (exposed for host-only tests):
// rank 0 sends fd_in to every other rank; *fd_out is the receiver's copy
// (rank 0: fd_in itself).
bool share_fd(int rank, int world, cmn_allgather_fn ag, void *user, int fd_in, int *fd_out,
              std::string &err);

}  // namespace cmn
