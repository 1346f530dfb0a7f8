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
    {  // views, quad_split and the overlap rules (ring.hpp:122-228)
        Modulus m7(101);
        Matrix M(6, 6, m7);
        MatView v = M.view();
        auto q = quad_split(v);
        if (q[3].ptr != &M.at(3, 3) || q[1].stride != 6) return 20;
        if (v.window(0, 0, 2, 2).overlaps(v.window(2, 2, 2, 2))) return 21;
        if (!v.window(1, 1, 2, 2).overlaps(v.window(0, 0, 2, 2))) return 22;
        if (!v.window(0, 1, 3, 1).overlaps(v.window(2, 0, 1, 2))) return 23;
        if (v.window(0, 2, 3, 1).overlaps(v.window(0, 3, 3, 3))) return 24;
        // brute force over every window pair of a 4x5 buffer
        Matrix N(4, 5, m7);
        MatView w = N.view();
        for (std::size_t r0 = 0; r0 < 4; ++r0)
            for (std::size_t c0 = 0; c0 < 5; ++c0)
                for (std::size_t r1 = 0; r1 < 4; ++r1)
                    for (std::size_t c1 = 0; c1 < 5; ++c1)
                        for (std::size_t h : {1, 2})
                            for (std::size_t wd : {1, 3}) {
                                if (r0 + h > 4 || c0 + wd > 5 || r1 + 2 > 4 || c1 + 2 > 5) continue;
                                MatView x = w.window(r0, c0, h, wd), y = w.window(r1, c1, 2, 2);
                                bool want = false;
                                for (std::size_t i = 0; i < h; ++i)
                                    for (std::size_t j = 0; j < wd; ++j)
                                        want |= r0 + i >= r1 && r0 + i < r1 + 2 && c0 + j >= c1 &&
                                                c0 + j < c1 + 2;
                                if (x.overlaps(y) != want || y.overlaps(x) != want) return 25;
                            }
        if (m7.reduce_i64(-1) != 100 || m7.reduce_u64(205) != 3) return 26;
        // the Workspace plug-ins (workspace.hpp:24-147)
        CostMeter meter;
        HeapWorkspace heap(&meter);
        heap.push_frame();
        heap.acquire(4, 4, 1, "X");
        heap.push_frame();
        heap.acquire(2, 2, 2, "Y");
        heap.pop_frame();
        heap.acquire(1, 3, 1, "Z");
        heap.pop_frame();
        if (meter.peak_extra_words != 20 || meter.total_alloc_words != 23 ||
            meter.live_extra_words != 0 || meter.alloc_log.size() != 3 ||
            meter.alloc_log[1].slot != "Y" || meter.alloc_log[1].depth != 2)
            return 27;
        Matrix D(8, 8, m7);
        QuadrantWorkspace qw(D.view());
        qw.push_frame();
        MatView t0 = qw.acquire(4, 4, 1, "X"), t1 = qw.acquire(4, 2, 1, "Y");
        qw.push_frame();
        MatView t2 = qw.acquire(2, 2, 2, "X");
        if (t0.ptr != &D.at(0, 0) || t1.ptr != &D.at(0, 4) || t2.ptr != &D.at(4, 4)) return 28;
        try {
            qw.acquire(2, 2, 2, "Y");
            qw.acquire(2, 2, 2, "Z");
            qw.acquire(1, 1, 2, "W");
            return 29;
        } catch (const workspace_error&) {
        }
        std::vector<Elem> chunk(10);
        BumpWorkspace bw(chunk.data(), chunk.size());
        bw.push_frame();
        bw.acquire(2, 3, 1, "X");
        try {
            bw.acquire(2, 3, 1, "Y");
            return 30;
        } catch (const workspace_error&) {
        }
        if (bw.high_water() != 6) return 31;
        // builtin headers and the blocked-variant grammar
        if (builtin("ip").contract != Contract::OverwriteBoth || !builtin("acc2").accumulating ||
            builtin("std2").square_only)
            return 33;
        if (!models::parse_blocked("blocked_acc_t3") || models::parse_blocked("blocked_acc_t") ||
            models::parse_blocked("blocked_acc_t2_acc2")->base != "acc2")
            return 34;
    }
    if (plan_only_mode) {
        std::printf("plan-only ok\n");
        return 0;
    }
    {  // the primitives on host views, executed on the device (ring.hpp:241-384)
        Modulus mod(kDefaultModulus);
        Matrix M(8, 8, mod);
        M.fill_random(5);
        Matrix M0 = M;
        auto q = quad_split(M.view());
        CostMeter meter;
        block_addsub(q[0], q[0], q[3], 1, mod.minus_one(), mod, &meter);  // exact alias of dst and a
        for (std::size_t i = 0; i < 4; ++i)
            for (std::size_t j = 0; j < 4; ++j)
                if (M.at(i, j) != mod.sub(M0.at(i, j), M0.at(i + 4, j + 4))) return 40;
        if (meter.adds != 16 || meter.mults != 0) return 41;
        try {
            block_addsub(M.view().window(1, 1, 4, 4), q[0], q[3], 1, 1, mod);
            return 42;
        } catch (const partial_overlap_error&) {
        }
        Matrix C(4, 4, mod), A(4, 4, mod), B(4, 4, mod);
        A.fill_random(6);
        B.fill_random(7);
        C.fill_random(8);
        Matrix want = C;
        for (std::size_t i = 0; i < 4; ++i)
            for (std::size_t j = 0; j < 4; ++j) {
                std::uint64_t acc = std::uint64_t(9) * C.at(i, j);
                for (std::size_t l = 0; l < 4; ++l) acc += std::uint64_t(3) * A.at(i, l) % 65521 * B.at(l, j);
                want.at(i, j) = static_cast<Elem>(acc % 65521);
            }
        classical_mul(C.view(), A.view(), B.view(), 3, 9, mod, &meter);
        if (!(C == want) || meter.classical_calls != 1) return 43;
        try {
            classical_mul(A.view(), A.view(), B.view(), 1, 0, mod);
            return 44;
        } catch (const alias_error&) {
        }
        block_scale_copy(q[1], q[2], mod.minus_one(), mod, &meter);
        for (std::size_t i = 0; i < 4; ++i)
            for (std::size_t j = 0; j < 4; ++j)
                if (M.at(i, j + 4) != mod.neg(M.at(i + 4, j))) return 45;
        std::printf("primitives ok\n");
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
        std::uint64_t logged = 0;  // alloc_log (meter.hpp:15-19) sums to the total
        for (const auto& e : meter.alloc_log) logged += e.words;
        if (logged != meter.total_alloc_words) return 12;
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
