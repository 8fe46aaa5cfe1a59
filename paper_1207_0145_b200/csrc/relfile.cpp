// relfile.cpp -- the reference's relation file format on the host side
// (magic "MPSMREL1", u64 n, n interleaved little-endian (key, payload) u64
// records; /root/reference/pkg/src/mpsm/bench.py:8-11,73-102).  Reading is
// parallel pread into the caller's (ideally pinned) buffer, so a file moves
// to the GPU as one H2D copy plus mpsm_deinterleave; host columns are split
// by the reading threads themselves, and writing is parallel pwrite of
// interleaved blocks (tools/relfile_bench.py).

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mpsm_b200.h"
#include "hostcpu.h"

namespace mpsm {
void set_error(const std::string& msg);
}

namespace {

constexpr char kMagic[8] = {'M', 'P', 'S', 'M', 'R', 'E', 'L', '1'};

struct Fd {
    int fd;
    explicit Fd(const char* path, int flags, int mode = 0644) : fd(::open(path, flags, mode)) {}
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

bool pread_all(int fd, char* dst, size_t bytes, off_t off) {
    while (bytes) {
        const ssize_t r = ::pread(fd, dst, bytes, off);
        if (r <= 0) return false;
        dst += r;
        off += r;
        bytes -= (size_t)r;
    }
    return true;
}

bool write_all(int fd, const char* src, size_t bytes) {
    while (bytes) {
        const ssize_t r = ::write(fd, src, bytes);
        if (r <= 0) return false;
        src += r;
        bytes -= (size_t)r;
    }
    return true;
}

bool pwrite_all(int fd, const char* src, size_t bytes, off_t off) {
    while (bytes) {
        const ssize_t r = ::pwrite(fd, src, bytes, off);
        if (r <= 0) return false;
        src += r;
        off += r;
        bytes -= (size_t)r;
    }
    return true;
}

// records [0, n) split over `threads` workers in contiguous ranges; fn(a, b)
// returns false on an I/O error
template <class F>
bool parallel_ranges(uint64_t n, int threads, F fn) {
    if (threads <= 0) threads = mpsm::usable_cores();
    const uint64_t per = std::max<uint64_t>((uint64_t)1 << 20, (n + threads - 1) / threads);
    std::vector<std::thread> pool;
    std::vector<char> ok;
    for (uint64_t a = 0; a < n; a += per) ok.push_back(1);
    size_t i = 0;
    for (uint64_t a = 0; a < n; a += per, ++i) {
        const uint64_t b = std::min(n, a + per);
        pool.emplace_back([&, a, b, i] { ok[i] = fn(a, b) ? 1 : 0; });
    }
    for (auto& t : pool) t.join();
    for (char c : ok)
        if (!c) return false;
    return true;
}

constexpr uint64_t kBlock = 1 << 16;  // records per thread-local block (1 MB)

}  // namespace

extern "C" int mpsm_relfile_header(const char* path, uint64_t* n, int64_t* bad_offset) {
    if (!path || !n) return MPSM_ERR_ARG;
    Fd f(path, O_RDONLY);
    if (f.fd < 0) {
        mpsm::set_error(std::string("cannot open ") + path + ": " + std::strerror(errno));
        return MPSM_ERR_IO;
    }
    struct stat st;
    if (::fstat(f.fd, &st) != 0) {
        mpsm::set_error(std::string("cannot stat ") + path);
        return MPSM_ERR_IO;
    }
    const uint64_t size = (uint64_t)st.st_size;
    char hdr[16] = {0};
    const size_t got = (size_t)std::min<uint64_t>(size, 16);
    if (got && !pread_all(f.fd, hdr, got, 0)) {
        mpsm::set_error(std::string("cannot read ") + path);
        return MPSM_ERR_IO;
    }
    // bench.py:88-99: magic, header length, exact record length
    if (size < 8 || std::memcmp(hdr, kMagic, 8) != 0) {
        if (bad_offset) *bad_offset = 0;
        mpsm::set_error(std::string("bad magic in ") + path);
        return MPSM_ERR_FORMAT;
    }
    if (size < 16) {
        if (bad_offset) *bad_offset = (int64_t)size;
        mpsm::set_error(std::string("truncated header in ") + path);
        return MPSM_ERR_FORMAT;
    }
    uint64_t cnt;
    std::memcpy(&cnt, hdr + 8, 8);  // little-endian host (x86-64 / aarch64)
    const unsigned __int128 expected = (unsigned __int128)16 + (unsigned __int128)16 * cnt;
    if ((unsigned __int128)size != expected) {
        if (bad_offset) *bad_offset = (int64_t)std::min<unsigned __int128>(size, expected);
        mpsm::set_error(std::string(path) + " declares " + std::to_string(cnt) + " tuples (" +
                        std::to_string((uint64_t)std::min<unsigned __int128>(expected, ~0ull)) +
                        " bytes) but has " + std::to_string(size));
        return MPSM_ERR_FORMAT;
    }
    *n = cnt;
    return MPSM_OK;
}

extern "C" int mpsm_relfile_read(const char* path, uint64_t n, void* dst, int threads) {
    if (!path || (!dst && n)) return MPSM_ERR_ARG;
    Fd f(path, O_RDONLY);
    if (f.fd < 0) {
        mpsm::set_error(std::string("cannot open ") + path + ": " + std::strerror(errno));
        return MPSM_ERR_IO;
    }
    const size_t bytes = (size_t)n * 16;
    if (threads <= 0) threads = mpsm::usable_cores();
    const size_t chunk = std::max<size_t>((size_t)64 << 20, (bytes + threads - 1) / threads);
    std::vector<std::thread> pool;
    std::vector<char> ok((bytes + chunk - 1) / chunk + 1, 1);
    size_t i = 0;
    for (size_t off = 0; off < bytes; off += chunk, ++i) {
        const size_t len = std::min(chunk, bytes - off);
        pool.emplace_back([&, off, len, i] { ok[i] = pread_all(f.fd, (char*)dst + off, len, (off_t)(16 + off)); });
    }
    for (auto& t : pool) t.join();
    for (char c : ok)
        if (!c) {
            mpsm::set_error(std::string("short read from ") + path);
            return MPSM_ERR_IO;
        }
    return MPSM_OK;
}

extern "C" int mpsm_relfile_read_columns(const char* path, uint64_t n, uint64_t* keys, uint64_t* pays, int threads) {
    if (!path || (n && (!keys || !pays))) return MPSM_ERR_ARG;
    Fd f(path, O_RDONLY);
    if (f.fd < 0) {
        mpsm::set_error(std::string("cannot open ") + path + ": " + std::strerror(errno));
        return MPSM_ERR_IO;
    }
    const bool ok = parallel_ranges(n, threads, [&](uint64_t a, uint64_t b) {
        std::vector<uint64_t> buf(2 * kBlock);
        for (uint64_t i = a; i < b; i += kBlock) {
            const size_t m = (size_t)std::min<uint64_t>(kBlock, b - i);
            if (!pread_all(f.fd, (char*)buf.data(), 16 * m, (off_t)(16 + 16 * i))) return false;
            for (size_t j = 0; j < m; ++j) {
                keys[i + j] = buf[2 * j];
                pays[i + j] = buf[2 * j + 1];
            }
        }
        return true;
    });
    if (!ok) {
        mpsm::set_error(std::string("short read from ") + path);
        return MPSM_ERR_IO;
    }
    return MPSM_OK;
}

extern "C" int mpsm_relfile_write(const char* path, const uint64_t* keys, const uint64_t* pays, uint64_t n) {
    if (!path || (n && (!keys || !pays))) return MPSM_ERR_ARG;
    Fd f(path, O_WRONLY | O_CREAT | O_TRUNC);
    if (f.fd < 0) {
        mpsm::set_error(std::string("cannot create ") + path + ": " + std::strerror(errno));
        return MPSM_ERR_IO;
    }
    char hdr[16];
    std::memcpy(hdr, kMagic, 8);
    std::memcpy(hdr + 8, &n, 8);
    if (!write_all(f.fd, hdr, 16)) return MPSM_ERR_IO;
    // interleaved blocks written at their offsets by parallel workers
    const bool ok = parallel_ranges(n, 0, [&](uint64_t a, uint64_t b) {
        std::vector<uint64_t> buf(2 * kBlock);
        for (uint64_t i = a; i < b; i += kBlock) {
            const size_t m = (size_t)std::min<uint64_t>(kBlock, b - i);
            for (size_t j = 0; j < m; ++j) {
                buf[2 * j] = keys[i + j];
                buf[2 * j + 1] = pays[i + j];
            }
            if (!pwrite_all(f.fd, (const char*)buf.data(), 16 * m, (off_t)(16 + 16 * i))) return false;
        }
        return true;
    });
    if (!ok) {
        mpsm::set_error(std::string("short write to ") + path);
        return MPSM_ERR_IO;
    }
    return MPSM_OK;
}
