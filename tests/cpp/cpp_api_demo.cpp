// C++ host program on the reference-shaped API (include/etdrd_b200/stepper.hpp).
// Usage: cpp_api_demo <scalar|system> dim n tau k0 k1 q family steps in.bin out.bin
//        cpp_api_demo errors
// in.bin holds U (and V) as raw float64, x-fastest; out.bin receives the result.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>

#include "etdrd_b200/stepper.hpp"

using namespace etdrd_b200;

static bool read_all(const char* path, double* dst, std::size_t n) {
    std::ifstream f(path, std::ios::binary);
    f.read(reinterpret_cast<char*>(dst), n * sizeof(double));
    return static_cast<std::size_t>(f.gcount()) == n * sizeof(double);
}

int main(int argc, char** argv) {
    if (argc == 2 && std::string(argv[1]) == "errors") {
        int ok = 0;
        try {
            (void)make_plan(unit_box_grid(2, 8), 0.0, 1.0, 1.0, PadeFamily::P02);
        } catch (const ConfigError&) { ++ok; }
        try {
            (void)unit_box_grid(3, 1);
        } catch (const ConfigError&) { ++ok; }
        const Grid g = unit_box_grid(2, 8);
        auto plan = make_plan(g, 0.01, 1.0, 1.0, PadeFamily::P02);
        StepperState st{4, 0.25, Field::zeros(g)};
        try {
            (void)advance(plan, st, DeviceSource{ETD_SRC_NAN, {}, true});
        } catch (const StepperAbort& e) {
            if (e.step == 4 && std::fabs(e.t - 0.25) < 1e-15) ++ok;
        }
        StepperState bad{0, 0.0, Field::zeros(unit_box_grid(2, 9))};
        try {
            (void)advance(plan, bad, DeviceSource::allen_cahn_cubic());
        } catch (const ConfigError&) { ++ok; }
        // make_plan's memory_cap_bytes: a plan above the cap is refused before allocating
        try {
            (void)make_plan(unit_box_grid(3, 64), 0.01, 1.0, 1.0, scheme_p02(), BackendKind::Spectral, 1 << 20);
        } catch (const MemoryGuardError&) { ++ok; }
        // RationalScheme values (rational.hpp:31-47): P02 one pole -1+i, P04 two
        const RationalScheme s2 = scheme_p02(), s4 = scheme_by_family(PadeFamily::P04);
        if (s2.for_ell(1).size() == 1 && s4.for_ell(3).size() == 2 && s2.terms[0][0].pole == std::complex<double>(-1, 1))
            ++ok;
        // ExactExpReference (stepper.cpp:259-295): a sine mode under f = 0 decays by
        // exactly e^{-tau lambda}, lambda the discrete eigenvalue (operators.cpp:43-53)
        {
            const int m = 32;
            const Grid ge = unit_box_grid(2, m);
            const double tau = 0.01, kap = 0.7, qq = 0.4, pi = 3.14159265358979323846, h = 1.0 / m;
            auto pe = make_plan(ge, tau, kap, qq, scheme_p02(), BackendKind::ExactExpReference);
            StepperState s0{0, 0.0, Field::zeros(ge)};
            for (int j = 0; j < m - 1; ++j)
                for (int i = 0; i < m - 1; ++i) s0.U.at(i, j) = std::sin(pi * (i + 1) * h) * std::sin(pi * (j + 1) * h);
            const StepperState s1 = etd2rkds_reference_step(pe, s0, DeviceSource{ETD_SRC_ZERO, {}, true});
            const double lam = 2.0 * (kap * 2.0 * (1.0 - std::cos(pi * h)) / (h * h) + qq / 2.0);
            double err = 0.0, mx = 0.0;
            for (std::size_t k = 0; k < s0.U.size(); ++k) {
                err = std::fmax(err, std::fabs(s1.U[k] - std::exp(-tau * lam) * s0.U[k]));
                mx = std::fmax(mx, std::fabs(s0.U[k]));
            }
            if (s1.n == 1 && err / mx <= 1e-12) ++ok;
            else std::printf("exact decay err %.3e\n", err / mx);
            try {
                (void)etd2rkds_step_2d(pe, s0, DeviceSource::allen_cahn_cubic());
            } catch (const ConfigError&) { ++ok; }
        }
        std::printf("errors ok=%d/8\n", ok);
        return ok == 8 ? 0 : 1;
    }
    if (argc != 12) {
        std::fprintf(stderr, "usage: see header\n");
        return 2;
    }
    const std::string kind = argv[1];
    const int dim = std::atoi(argv[2]), n = std::atoi(argv[3]), steps = std::atoi(argv[9]);
    const double tau = std::atof(argv[4]), k0 = std::atof(argv[5]), k1 = std::atof(argv[6]), q = std::atof(argv[7]);
    const PadeFamily fam = std::atoi(argv[8]) ? PadeFamily::P04 : PadeFamily::P02;
    const Grid g = unit_box_grid(dim, n + 1);
    const std::size_t N = g.total_interior();
    if (kind == "scalar") {
        auto plan = make_plan(g, tau, k0, q, fam);
        StepperState st{0, 0.0, Field::zeros(g)};
        if (!read_all(argv[10], st.U.data(), N)) return 3;
        for (int s = 0; s < steps; ++s) st = advance(plan, st, DeviceSource::allen_cahn_cubic());
        std::ofstream(argv[11], std::ios::binary).write(reinterpret_cast<const char*>(st.U.data()), N * 8);
        std::printf("n=%ld t=%.6f\n", st.n, st.t);
    } else {
        auto plan = make_system_plan(g, tau, k0, k1, q, fam);
        SystemState st{0, 0.0, Field::zeros(g), Field::zeros(g)};
        std::vector<double> buf(2 * N);
        if (!read_all(argv[10], buf.data(), 2 * N)) return 3;
        std::memcpy(st.U.data(), buf.data(), N * 8);
        std::memcpy(st.V.data(), buf.data() + N, N * 8);
        st = etd2rkds_step_system(plan, st, DeviceSource::fhn_cubic(), steps);
        std::ofstream o(argv[11], std::ios::binary);
        o.write(reinterpret_cast<const char*>(st.U.data()), N * 8);
        o.write(reinterpret_cast<const char*>(st.V.data()), N * 8);
        std::printf("n=%ld t=%.6f\n", st.n, st.t);
    }
    return 0;
}
