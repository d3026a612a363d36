// C++ host program on the reference-shaped API (include/etdrd_b200/stepper.hpp).
// Usage: cpp_api_demo <scalar|system> dim n tau k0 k1 q family steps in.bin out.bin
//        cpp_api_demo errors
// in.bin holds U (and V) as raw float64, x-fastest; out.bin receives the result.
#include <cmath>
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
        std::printf("errors ok=%d/4\n", ok);
        return ok == 4 ? 0 : 1;
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
