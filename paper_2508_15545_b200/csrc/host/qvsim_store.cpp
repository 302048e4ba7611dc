// qvsim_store.cpp — QVSV state files and the file-backed GPU apply_circuit.
//
// The file format is the reference's (store.hpp:24-29): a 32-byte header
// followed by the amplitudes, so stores are interchangeable with the
// reference's BlockStore (tests/test_store.py checks both directions). The GPU
// path replaces the reference's per-gate block streaming with one
// file -> HBM load, the whole circuit on the device, and one HBM -> file store,
// each in large pinned chunks double-buffered against the PCIe copies.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <exception>
#include <mutex>
#include <thread>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>

#include "qvsim_gpu.hpp"

namespace qvsim {

namespace {

constexpr std::uint64_t kHeaderBytes = 32;
constexpr std::uint32_t kVersion = 1;
constexpr std::uint64_t kChunkAmps = 1ull << 24;  // 256 MiB pinned staging chunks

[[noreturn]] void io_fail(const std::string &what, const std::string &path) {
    throw IoError(what + " '" + path + "': " + std::strerror(errno));
}

void put_le(unsigned char *p, std::uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}

std::uint64_t get_le(const unsigned char *p, int bytes) {
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= std::uint64_t{p[i]} << (8 * i);
    return v;
}

void check_shape(std::uint32_t n, std::uint64_t block_amps) {
    if (n < 1 || n > kMaxQubits)
        throw ValidationError("n_qubits must be in [1, " + std::to_string(kMaxQubits) + "], got " + std::to_string(n));
    if (block_amps == 0 || (block_amps & (block_amps - 1)))
        throw ValidationError("block_amps must be a power of two, got " + std::to_string(block_amps));
    if (block_amps > (std::uint64_t{1} << n))
        throw ValidationError("block_amps " + std::to_string(block_amps) + " exceeds state length 2^" +
                              std::to_string(n));
}

void pread_all(int fd, void *dst, std::uint64_t bytes, std::uint64_t off, const std::string &path) {
    auto *p = static_cast<char *>(dst);
    while (bytes) {
        const ssize_t r = ::pread(fd, p, std::min<std::uint64_t>(bytes, 1ull << 30), (off_t)off);
        if (r < 0) {
            if (errno == EINTR) continue;
            io_fail("cannot read", path);
        }
        if (r == 0) throw FormatError("unexpected end of file in '" + path + "'");
        p += r;
        off += (std::uint64_t)r;
        bytes -= (std::uint64_t)r;
    }
}

void pwrite_all(int fd, const void *src, std::uint64_t bytes, std::uint64_t off, const std::string &path) {
    auto *p = static_cast<const char *>(src);
    while (bytes) {
        const ssize_t w = ::pwrite(fd, p, std::min<std::uint64_t>(bytes, 1ull << 30), (off_t)off);
        if (w < 0) {
            if (errno == EINTR) continue;
            io_fail("cannot write", path);
        }
        p += w;
        off += (std::uint64_t)w;
        bytes -= (std::uint64_t)w;
    }
}

// Two pinned staging buffers from libqvg (cudaHostAlloc), freed on scope exit.
// Two page-locked staging buffers. Pinning 512 MiB costs ~0.3 s, more than
// moving a 16 GiB state through them, so released buffers are kept in a
// process-wide pool and reused by the next call (held until exit).
class Pinned {
  public:
    void *buf[2] = {nullptr, nullptr};
    explicit Pinned(std::uint64_t bytes) : bytes_(bytes) {
        std::lock_guard<std::mutex> lock(mu());
        auto &free = pool();
        for (auto &b : buf) {
            auto it = std::find_if(free.begin(), free.end(), [&](const auto &e) { return e.first == bytes; });
            if (it != free.end()) {
                b = it->second;
                free.erase(it);
            } else {
                check_status(qvg_host_alloc(bytes, &b));
            }
        }
    }
    ~Pinned() {
        std::lock_guard<std::mutex> lock(mu());
        for (auto *b : buf)
            if (b) pool().push_back({bytes_, b});
    }
    Pinned(const Pinned &) = delete;
    Pinned &operator=(const Pinned &) = delete;

  private:
    std::uint64_t bytes_;
    static std::mutex &mu() {
        static std::mutex m;
        return m;
    }
    static std::vector<std::pair<std::uint64_t, void *>> &pool() {
        static auto *p = new std::vector<std::pair<std::uint64_t, void *>>();  // never destroyed: pinned until exit
        return *p;
    }
};

}  // namespace

StateStore::StateStore(int fd, std::string path, std::uint32_t n, std::uint64_t block_amps)
    : fd_(fd), path_(std::move(path)), n_(n), block_amps_(block_amps) {}

StateStore::StateStore(StateStore &&o) noexcept : fd_(o.fd_), path_(std::move(o.path_)), n_(o.n_), block_amps_(o.block_amps_) {
    o.fd_ = -1;
}

StateStore &StateStore::operator=(StateStore &&o) noexcept {
    if (this != &o) {
        if (fd_ >= 0) ::close(fd_);
        fd_ = o.fd_;
        path_ = std::move(o.path_);
        n_ = o.n_;
        block_amps_ = o.block_amps_;
        o.fd_ = -1;
    }
    return *this;
}

StateStore::~StateStore() {
    if (fd_ >= 0) ::close(fd_);
}

StateStore StateStore::create(const std::string &path, std::uint32_t n, std::uint64_t block_amps, bool overwrite) {
    check_shape(n, block_amps);
    const int fd = ::open(path.c_str(), O_RDWR | O_CREAT | (overwrite ? O_TRUNC : O_EXCL), 0644);
    if (fd < 0) {
        if (errno == EEXIST) throw IoError("file exists (pass overwrite to replace): '" + path + "'");
        io_fail("cannot create", path);
    }
    StateStore s(fd, path, n, block_amps);
    unsigned char hdr[kHeaderBytes] = {'Q', 'V', 'S', 'V'};
    put_le(hdr + 4, kVersion, 4);
    put_le(hdr + 8, n, 4);
    put_le(hdr + 12, block_amps, 8);
    pwrite_all(fd, hdr, kHeaderBytes, 0, path);
    // full length; the unwritten payload reads back as zeros, i.e. |0...0>
    // once amplitude 0 is set
    if (::ftruncate(fd, (off_t)(kHeaderBytes + (16ull << n))) != 0) io_fail("cannot size", path);
    const double one[2] = {1.0, 0.0};
    pwrite_all(fd, one, sizeof(one), kHeaderBytes, path);
    return s;
}

StateStore StateStore::open(const std::string &path) {
    const int fd = ::open(path.c_str(), O_RDWR);
    if (fd < 0) io_fail("cannot open", path);
    struct stat st {};
    if (::fstat(fd, &st) != 0) {
        ::close(fd);
        io_fail("cannot stat", path);
    }
    unsigned char hdr[kHeaderBytes];
    try {
        if ((std::uint64_t)st.st_size < kHeaderBytes)
            throw FormatError("file is shorter than the " + std::to_string(kHeaderBytes) + "-byte header");
        pread_all(fd, hdr, kHeaderBytes, 0, path);
        if (std::memcmp(hdr, "QVSV", 4) != 0) throw FormatError("bad magic in '" + path + "'");
        if (get_le(hdr + 4, 4) != kVersion)
            throw FormatError("unsupported version " + std::to_string(get_le(hdr + 4, 4)));
        const auto n = (std::uint32_t)get_le(hdr + 8, 4);
        const std::uint64_t ba = get_le(hdr + 12, 8);
        check_shape(n, ba);
        if ((std::uint64_t)st.st_size != kHeaderBytes + (16ull << n))
            throw FormatError("file length " + std::to_string(st.st_size) +
                              " does not match header-implied size " + std::to_string(kHeaderBytes + (16ull << n)));
        return StateStore(fd, path, n, ba);
    } catch (...) {
        ::close(fd);
        throw;
    }
}

namespace {

// Large file transfers are split over host threads: a tmpfs / page-cache copy
// is memcpy-bound at ~5 GB/s per thread, far below PCIe, and it dominates the
// file-level drop-in (tools/store_e2e.py).
template <class F> void split_io(std::uint64_t bytes, F &&piece) {
    constexpr std::uint64_t kMinPiece = 4ull << 20;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::uint64_t parts = std::min<std::uint64_t>({std::uint64_t{16}, hw, std::max<std::uint64_t>(1, bytes / kMinPiece)});
    if (parts <= 1) {
        piece(0, bytes);
        return;
    }
    const std::uint64_t step = (bytes / parts + 15) & ~std::uint64_t{15};
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errors(parts);
    for (std::uint64_t i = 0; i < parts; ++i) {
        const std::uint64_t a = std::min(bytes, i * step), b = std::min(bytes, a + step);
        if (a >= b) break;
        pool.emplace_back([&, i, a, b] {
            try {
                piece(a, b - a);
            } catch (...) {
                errors[i] = std::current_exception();
            }
        });
    }
    for (auto &t : pool) t.join();
    for (auto &e : errors)
        if (e) std::rethrow_exception(e);
}

}  // namespace

void StateStore::read(amp_t *out, std::uint64_t offset, std::uint64_t count) const {
    if (offset > n_amps() || count > n_amps() - offset) throw ValidationError("amplitude range out of range");
    auto *dst = reinterpret_cast<unsigned char *>(out);
    split_io(count * 16, [&](std::uint64_t at, std::uint64_t len) {
        pread_all(fd_, dst + at, len, kHeaderBytes + offset * 16 + at, path_);
    });
}

void StateStore::write(const amp_t *in, std::uint64_t offset, std::uint64_t count) {
    if (offset > n_amps() || count > n_amps() - offset) throw ValidationError("amplitude range out of range");
    const auto *src = reinterpret_cast<const unsigned char *>(in);
    const std::uint64_t bytes = count * 16, start = kHeaderBytes + offset * 16;
    // Concurrent pwrite()s to one file serialise on the inode lock, so large
    // writes go through a shared mapping that many threads fill at once
    // (5.9 -> tens of GB/s on tmpfs; tools/store_e2e.py). The file already
    // has its full length (create() sizes it).
    if (bytes >= (64ull << 20)) {
        const std::uint64_t page = (std::uint64_t)::sysconf(_SC_PAGESIZE);
        const std::uint64_t map_off = start & ~(page - 1), lead = start - map_off;
        void *m = ::mmap(nullptr, lead + bytes, PROT_WRITE, MAP_SHARED, fd_, (off_t)map_off);
        if (m != MAP_FAILED) {
            unsigned char *dst = static_cast<unsigned char *>(m) + lead;
            split_io(bytes, [&](std::uint64_t at, std::uint64_t len) { std::memcpy(dst + at, src + at, len); });
            if (::munmap(m, lead + bytes) != 0) io_fail("munmap failed on", path_);
            return;
        }
    }
    split_io(bytes, [&](std::uint64_t at, std::uint64_t len) { pwrite_all(fd_, src + at, len, start + at, path_); });
}

amp_t StateStore::amplitude(std::uint64_t index) const {
    if (index >= n_amps()) throw ValidationError("amplitude index " + std::to_string(index) + " out of range");
    amp_t a;
    read(&a, index, 1);
    return a;
}

double StateStore::norm() const {
    double sum = 0.0, carry = 0.0;
    std::vector<amp_t> buf(std::min<std::uint64_t>(n_amps(), kChunkAmps));
    for (std::uint64_t off = 0; off < n_amps(); off += buf.size()) {
        const std::uint64_t c = std::min<std::uint64_t>(buf.size(), n_amps() - off);
        read(buf.data(), off, c);
        for (std::uint64_t i = 0; i < c; ++i) {
            const double term = std::norm(buf[i]) - carry;
            const double next = sum + term;
            carry = (next - sum) - term;
            sum = next;
        }
    }
    return std::sqrt(sum);
}

void StateStore::sync() const {
    if (::fdatasync(fd_) != 0) io_fail("sync failed on", path_);
}

void apply_circuit(StateStore &store, const Circuit &circuit, const RunConfig &config, Metrics &metrics,
                   int device) {
    if (circuit.n_qubits != store.n_qubits())
        throw ValidationError("circuit is for " + std::to_string(circuit.n_qubits) + " qubits, store holds " +
                              std::to_string(store.n_qubits()));
    if (config.strategy != Strategy::gpu)
        throw ValidationError(std::string("strategy '") + strategy_tag(config.strategy) +
                              "' is the reference's CPU engine; this build provides 'gpu'");
    if (const auto v = validate_circuit(circuit); !v.empty())
        throw ValidationError("invalid circuit: op " + std::to_string(v.front().op_index) + ": " + v.front().message);
    const double before = metrics.wall_ms;
    const auto t0 = std::chrono::steady_clock::now();
    // Out-of-core when asked, or when the state does not fit next to the
    // workspace: two HBM windows of the largest power of two that fits 40% of
    // free memory each (the paper's disk tier on the GPU).
    std::uint32_t w = config.window_qubits;
    if (w == 0) {
        std::uint64_t free_b = 0, total_b = 0;
        check_status(qvg_device_memory(device, &free_b, &total_b));
        if ((16ull << store.n_qubits()) > free_b * 9 / 10) {
            w = 4;
            while ((16ull << (w + 1)) <= free_b * 4 / 10 && w + 1 < store.n_qubits()) ++w;
        }
    }
    if (w > 0) {
        const std::vector<qvg_gate> gates = to_gates(circuit);
        auto io = [](void *user, std::uint64_t off, std::uint64_t cnt, void *buf, int write) -> int {
            auto *st = static_cast<StateStore *>(user);
            try {
                if (write) st->write(static_cast<const amp_t *>(buf), off, cnt);
                else st->read(static_cast<amp_t *>(buf), off, cnt);
                return 0;
            } catch (...) {
                return 1;
            }
        };
        qvg_stats s{};
        check_status(qvg_apply_stream(io, &store, store.n_qubits(), 128, device, w, gates.data(), gates.size(), &s));
        metrics.strategy = strategy_tag(config.strategy);
        metrics.gates_applied += s.gates_applied;
        metrics.traversals += s.passes;
        metrics.fused_passes += s.fused_passes;
        metrics.bytes_moved += s.bytes_moved;
        metrics.bytes_read += s.exchange_bytes / 2;
        metrics.bytes_written += s.exchange_bytes / 2;
        metrics.exchanges += s.exchanges;  // whole-state round trips (segments)
        metrics.blocks_read += s.exchange_bytes / 2 / (store.block_amps() * 16);
        metrics.blocks_written += s.exchange_bytes / 2 / (store.block_amps() * 16);
        metrics.peak_cache_bytes = std::max<std::uint64_t>(metrics.peak_cache_bytes, 2 * (16ull << w));
        metrics.wall_ms =
            before + std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return;
    }
    StateVector sv = StateVector::create(store.n_qubits(), 128, device);
    const std::uint64_t total = store.n_amps();
    const std::uint64_t chunk = std::min<std::uint64_t>(total, kChunkAmps);
    Pinned pin(chunk * 16);
    const auto t_setup = std::chrono::steady_clock::now();
    // file -> pinned[i%2] -> HBM; the read of chunk i+1 overlaps the H2D of
    // chunk i. The buffer a read refills was last used by the H2D two chunks
    // back, which the previous iteration's sync already waited for.
    std::uint64_t k = 0;
    for (std::uint64_t off = 0; off < total; off += chunk, ++k) {
        const std::uint64_t c = std::min(chunk, total - off);
        store.read(static_cast<amp_t *>(pin.buf[k % 2]), off, c);
        sv.sync();  // the H2D of the previous chunk (it ran during this read)
        check_status(qvg_load_async(sv.handle(), pin.buf[k % 2], off, c));
        metrics.bytes_read += c * 16;
    }
    const auto t_in = std::chrono::steady_clock::now();
    RunConfig dev_cfg = config;
    dev_cfg.sync = false;
    apply_circuit(sv, circuit, dev_cfg, metrics);
    if (std::getenv("QVG_TRACE")) {
        sv.sync();
        std::fprintf(stderr, "[qvg] store apply: setup %.1f ms, file->HBM %.1f ms, gates %.1f ms\n",
                     std::chrono::duration<double, std::milli>(t_setup - t0).count(),
                     std::chrono::duration<double, std::milli>(t_in - t_setup).count(),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_in).count());
    }
    // HBM -> pinned[i%2] -> file; the D2H of chunk i+1 overlaps the write of chunk i
    k = 0;
    std::uint64_t pending_off = 0, pending_c = 0;
    for (std::uint64_t off = 0; off < total; off += chunk, ++k) {
        const std::uint64_t c = std::min(chunk, total - off);
        check_status(qvg_read_async(sv.handle(), pin.buf[k % 2], off, c));
        if (pending_c) {
            store.write(static_cast<const amp_t *>(pin.buf[(k + 1) % 2]), pending_off, pending_c);
            metrics.bytes_written += pending_c * 16;
        }
        sv.sync();
        pending_off = off;
        pending_c = c;
    }
    if (pending_c) {
        store.write(static_cast<const amp_t *>(pin.buf[(k + 1) % 2]), pending_off, pending_c);
        metrics.bytes_written += pending_c * 16;
    }
    metrics.blocks_read += store.n_blocks();
    metrics.blocks_written += store.n_blocks();
    metrics.wall_ms = before + std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

std::vector<std::pair<std::uint64_t, amp_t>> top_amplitudes(const StateStore &store, std::size_t k) {
    std::vector<std::pair<std::uint64_t, amp_t>> out;
    if (k == 0) return out;
    struct E {
        double p;
        std::uint64_t i;
        amp_t a;
    };
    auto better = [](const E &x, const E &y) { return x.p != y.p ? x.p > y.p : x.i < y.i; };
    std::priority_queue<E, std::vector<E>, decltype(better)> heap(better);
    std::vector<amp_t> buf(std::min<std::uint64_t>(store.n_amps(), kChunkAmps));
    for (std::uint64_t off = 0; off < store.n_amps(); off += buf.size()) {
        const std::uint64_t c = std::min<std::uint64_t>(buf.size(), store.n_amps() - off);
        store.read(buf.data(), off, c);
        for (std::uint64_t j = 0; j < c; ++j) {
            const E e{std::norm(buf[j]), off + j, buf[j]};
            if (heap.size() < k) heap.push(e);
            else if (better(e, heap.top())) {
                heap.pop();
                heap.push(e);
            }
        }
    }
    std::vector<E> all;
    while (!heap.empty()) {
        all.push_back(heap.top());
        heap.pop();
    }
    std::sort(all.begin(), all.end(), better);
    for (const E &e : all) out.emplace_back(e.i, e.a);
    return out;
}

}  // namespace qvsim
