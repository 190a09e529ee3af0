// libm_pow_host.cu -- host side of libm_pow.cuh: find glibc's pow tables inside the libm
// loaded by this process, check the restatement bitwise against ::pow, and hand the table
// image to the device (see libm_pow.cuh for why the boundary-state pow must round as the
// reference's libm does, disc_euler.cpp:179-180,187).
#include <link.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fnlh_b200.h"
#include "libm_pow.cuh"

namespace fnlh {
namespace {

struct Seg {
    const unsigned char* p;
    std::size_t n;
};

int collect(struct dl_phdr_info* info, size_t, void* data) {
    const char* name = info->dlpi_name ? info->dlpi_name : "";
    if (!std::strstr(name, "libm.so")) return 0;
    auto* segs = static_cast<std::vector<Seg>*>(data);
    for (int h = 0; h < info->dlpi_phnum; ++h) {
        const ElfW(Phdr)& ph = info->dlpi_phdr[h];
        if (ph.p_type == PT_LOAD && (ph.p_flags & PF_R) && !(ph.p_flags & PF_W))
            segs->push_back({reinterpret_cast<const unsigned char*>(info->dlpi_addr + ph.p_vaddr), ph.p_memsz});
    }
    return 0;
}

uint64_t u64(const unsigned char* p) {
    uint64_t u;
    std::memcpy(&u, p, 8);
    return u;
}
double f64(const unsigned char* p) {
    double d;
    std::memcpy(&d, p, 8);
    return d;
}

// pow_log_data: ln2hi, ln2lo (the usual 2-part split of ln 2) and A[0] = -1/2, then 6
// further coefficients and the 128 x {invc, pad, logc, logctail} table.
// exp_data: invln2N = 128/ln2 and shift = 1.5 * 2^52 lead the header, ln2/128 split in
// two, the 4 coefficients C2..C5; the table {tail, sbits} x 128 starts with (0, bits(1.0)),
// and entry j has sbits + (j << 45) = bits(2^(j/128)) to within an ulp.
bool locate(double* T) {
    std::vector<Seg> segs;
    dl_iterate_phdr(collect, &segs);
    const unsigned char *logp = nullptr, *expp = nullptr, *tabp = nullptr;
    for (const Seg& s : segs) {
        for (std::size_t o = 0; o + 8 * 24 <= s.n; o += 8) {
            const unsigned char* p = s.p + o;
            if (!logp && u64(p) == 0x3fe62e42fefa3800ull && u64(p + 8) == 0x3d2ef35793c76730ull &&
                f64(p + 16) == -0.5)
                logp = p;
            if (!expp && u64(p) == 0x40671547652b82feull && u64(p + 8) == 0x4338000000000000ull)
                expp = p;
            if (!tabp && u64(p) == 0 && u64(p + 8) == 0x3ff0000000000000ull && o + 8 * 256 <= s.n) {
                bool ok = true;
                for (int j = 1; j < 128 && ok; ++j) {
                    const uint64_t sb = u64(p + 16 * j + 8) + ((uint64_t)j << 45);
                    const uint64_t want = pw_bits(std::exp2(j / 128.0));
                    ok = (sb > want ? sb - want : want - sb) <= 1;
                }
                if (ok) tabp = p;
            }
        }
    }
    if (!logp || !expp || !tabp) return false;
    std::memcpy(T + kPowLogHdr, logp, 9 * 8);
    std::memcpy(T + kPowLogTab, logp + 9 * 8, 512 * 8);
    std::memcpy(T + kPowExpHdr, expp, 4 * 8);
    // C2..C5 follow the two ln2/N parts; they are the next four doubles of the header
    std::memcpy(T + kPowExpHdr + 4, expp + 4 * 8, 4 * 8);
    std::memcpy(T + kPowExpTab, tabp, 256 * 8);
    return true;
}

// a fixed argument sample: the boundary-state exponents gamma/(gamma-1) and 1/gamma over
// temperature / pressure ratios around 1, and a log-uniform sweep of both arguments
bool validate(const double* T, long long* checked) {
    uint64_t s = 0x9e3779b97f4a7c15ull;
    auto next = [&] {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        return (double)(s >> 11) * 0x1p-53;
    };
    long long n = 0;
    auto one = [&](double x, double y) {
        double r;
        ++n;
        if (!pow_libm_main(T, x, y, &r)) return true;  // outside the restated path: cr_pow
        const double g = std::pow(x, y);
        return pw_bits(r) == pw_bits(g);
    };
    const double ys[] = {1.4 / 0.4, 1.0 / 1.4, 1.3 / 0.3, 1.0 / 1.3, 3.5, 0.5, -1.5, 2.0 / 7.0};
    for (double y : ys)
        for (int k = 0; k < 40000; ++k)
            if (!one(0.8 + 0.4 * next(), y)) return false;
    for (int k = 0; k < 100000; ++k) {
        const double x = std::exp2(-60.0 + 120.0 * next());
        const double y = (next() < 0.5 ? -1.0 : 1.0) * std::exp2(-8.0 + 12.0 * next());
        if (!one(x, y)) return false;
    }
    if (!one(1.0, 3.5) || !one(1.0 + 0x1p-52, 3.5) || !one(1.0 - 0x1p-53, 1.0 / 1.4)) return false;
    *checked = n;
    return true;
}

struct PowState {
    std::vector<double> T;
    bool ok = false;
    long long checked = 0;
    std::string why;
};

PowState& state() {
    static PowState st;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("FNLH_POW");
        if (env && std::string(env) == "cr") {
            st.why = "FNLH_POW=cr";
            return;
        }
        st.T.assign(kPowTabDoubles, 0.0);
        if (!locate(st.T.data())) {
            st.why = "glibc pow tables not found in the loaded libm";
            return;
        }
        if (!validate(st.T.data(), &st.checked)) {
            st.why = "restated pow differs from the host libm's";
            return;
        }
        st.ok = true;
        st.why = "glibc pow restated (" + std::to_string(st.checked) + " arguments bitwise equal to ::pow)";
    });
    return st;
}

}  // namespace

// the table image for the device, or nullptr (correctly rounded pow)
const double* libm_pow_tables() {
    PowState& st = state();
    return st.ok ? st.T.data() : nullptr;
}

}  // namespace fnlh

extern "C" {

int fnlh_pow_mode(void) { return fnlh::state().ok ? 0 : 1; }

const char* fnlh_pow_mode_info(void) { return fnlh::state().why.c_str(); }

double fnlh_pow(double x, double y) { return fnlh::bc_pow(fnlh::libm_pow_tables(), x, y); }

}  // extern "C"
