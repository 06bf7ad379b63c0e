// TEST: the pair introsort (parsa_stdsort_pairs.hpp) orders every tie-heavy
// random input exactly like psa_std_sort (parsa_stdsort.h) — and like
// libstdc++'s std::sort itself on the (key, id) vertices; so does its task
// form (sort_tasks, the device's parallel exact sort).
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "parsa_stdsort_pairs.hpp"

int main() {
    std::mt19937_64 rng(12345);
    long bad = 0, cases = 0;
    for (int m : {1, 2, 3, 5, 16, 17, 18, 33, 34, 64, 101, 257, 500, 501, 1001, 4001}) {
        for (int rep = 0; rep < 300; ++rep) {
            const int distinct = 1 + static_cast<int>(rng() % (m + 1));
            std::vector<double> key(m);
            for (auto& k : key) k = static_cast<double>(rng() % distinct) * 0.5;
            std::vector<int> ids(m);
            for (int i = 0; i < m; ++i) ids[i] = static_cast<int>(rng() % 1000000) * 0 + i;
            std::shuffle(ids.begin(), ids.end(), rng);
            std::vector<int> a = ids;
            psa_std_sort(a.data(), m, key.data());
            std::vector<psa_sort::KeyId> p(m);
            for (int i = 0; i < m; ++i) p[i] = {key[ids[i]], ids[i], 0};
            std::vector<psa_sort::KeyId> t = p;
            psa_sort::sort(p.data(), m);
            psa_sort::sort_tasks(t.data(), m);
            struct V { double f; int id; };
            std::vector<V> s(m);
            for (int i = 0; i < m; ++i) s[i] = {key[ids[i]], ids[i]};
            std::sort(s.begin(), s.end(), [](const V& x, const V& y) { return x.f < y.f; });
            for (int i = 0; i < m; ++i)
                if (a[i] != p[i].id || s[i].id != a[i] || t[i].id != a[i]) {
                    ++bad;
                    break;
                }
            ++cases;
        }
    }
    std::printf("stdsort pairs check: %ld cases, %ld mismatches\n", cases, bad);
    return bad ? 1 : 0;
}
