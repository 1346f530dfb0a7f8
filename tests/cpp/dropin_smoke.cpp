// Drop-in smoke test: reference-style code compiled against include/winomem_b200.hpp.
// --plan-only: host planning only (no GPU); otherwise also runs on the device and
// checks C against a naive product.
#include <cstdio>
#include <cstring>
#include <sstream>

#include "winomem_b200.hpp"

using namespace winomem;

int main(int argc, char** argv) {
    const bool plan_only_mode = argc > 1 && std::strcmp(argv[1], "--plan-only") == 0;
    // the reference's own closed forms (test_models.cpp:22-43)
    if (models::expected_costs("std2", 4, 4, 4, 1).peak_extra_words != 10) return 1;
    if (models::expected_costs("acc2", 32, 32, 32, 1).peak_extra_words != 682) return 2;
    CostReport r = plan_only("std2", 1024, 1024, 1024, {1, 0, 128});
    if (r.peak_extra_words != 688128 || r.mults != 719323136ull) return 3;
    try {
        plan_only("ip", 4, 8, 4);
        return 4;
    } catch (const shape_error&) {
    }
    // schedule DSL: every builtin renders and parses back to itself
    for (const auto& name : builtin_names()) {
        Schedule b = builtin(name);
        Schedule t = parse_schedule(render_schedule(b));
        if (!t.builtin_match || t.text != b.text || t.name != name) return 5;
    }
    try {
        parse_schedule("1: S1 = A21 + NOPE @ X\n");
        return 6;
    } catch (const unknown_slot_error&) {
    }
    {  // matrix file formats round trip (ring.hpp:386-449)
        Modulus m7(101);
        Matrix a(3, 4, m7);
        a.fill_random(9);
        std::stringstream t, b;
        write_text(a, t);
        write_binary(a, b);
        if (!(read_text(t) == a) || !(read_binary(b) == a)) return 7;
        std::stringstream bad("2 2 7\n1 2 3 9\n");
        try {
            read_text(bad);
            return 8;
        } catch (const io_error&) {
        }
    }
    if (plan_only_mode) {
        std::printf("plan-only ok\n");
        return 0;
    }
    Modulus mod(kDefaultModulus);
    for (const char* v : {"std2", "acc2", "ip", "ipmm"}) {
        const bool acc = variant_accumulates(v);
        Matrix A(64, 64, mod), B(64, 64, mod), C(64, 64, mod);
        A.fill_random(1);
        B.fill_random(2);
        if (acc) C.fill_random(3);
        Matrix want = C;
        for (std::size_t i = 0; i < 64; ++i)
            for (std::size_t j = 0; j < 64; ++j) {
                std::uint64_t s = acc ? C.at(i, j) : 0;
                for (std::size_t l = 0; l < 64; ++l) s += std::uint64_t(A.at(i, l)) * B.at(l, j) % 65521;
                want.at(i, j) = static_cast<Elem>(s % 65521);
            }
        Matrix C0 = C;
        CostMeter meter;
        run_variant(v, A, B, C, {1, acc ? 1u : 0u, 8}, &meter);
        if (!(C == want)) {
            std::printf("%s mismatch\n", v);
            return 10;
        }
        if (std::strcmp(v, "ipmm") != 0) {  // the same schedule as DSL text
            Matrix A2(64, 64, mod), B2(64, 64, mod);
            A2.fill_random(1);
            B2.fill_random(2);
            CostReport pr = run_parsed_schedule(parse_schedule(builtin(v).text), A2, B2, C0,
                                                {1, acc ? 1u : 0u, 8});
            if (!(C0 == want) || pr.mults != meter.mults || pr.peak_extra_words != meter.peak_extra_words) {
                std::printf("%s parsed mismatch\n", v);
                return 11;
            }
        }
        std::printf("%s ok peak=%llu launches=%llu\n", v, (unsigned long long)meter.peak_extra_words,
                    (unsigned long long)meter.launches);
    }
    return 0;
}
