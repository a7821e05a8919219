// field_eval_b200.cpp — the reference's evaluate() (field_eval.hpp:27) on the
// B200 potential kernel K3 (bw_potential). Links in place of
// proj/src/field_eval.cpp; a target within one panel diameter throws
// NearFieldError as field_eval.cpp:12-13 does.
#include <mutex>
#include <vector>

#include "biewos/field_eval.hpp"
#include "biewos_b200_bridge.hpp"

namespace biewos {

namespace {
std::mutex g_call;
}

Real evaluate(const BoundaryData& data, const Vec3& x) {
    std::vector<double> panels;
    panels.reserve(9 * data.panels.size());
    for (const BoundaryPanel& p : data.panels)
        panels.insert(panels.end(), {p.point.x(), p.point.y(), p.point.z(), p.normal.x(),
                                     p.normal.y(), p.normal.z(), p.area, p.u, p.dudn});
    const double t[3] = {x.x(), x.y(), x.z()};
    double u = 0;
    bw_status st;
    {
        std::lock_guard<std::mutex> lk(g_call);
        st = bw_potential(b200::context(), panels.data(), static_cast<int64_t>(data.panels.size()),
                          t, 1, &u, nullptr);
    }
    b200::check(st);
    return u;
}

} // namespace biewos
