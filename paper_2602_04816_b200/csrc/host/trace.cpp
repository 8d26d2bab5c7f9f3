// JSONL export of the measured event trace (reference proj/src/trace.cpp:56-79
// schema, plus t_start_us / t_end_us).
#include "hlm/trace.hpp"

#include <cstdio>
#include <sstream>

namespace hlm {
inline namespace b200 {

const char* stream_name(StreamId s) {
    switch (s) {
        case StreamId::H2D: return "h2d";
        case StreamId::Compute: return "compute";
        case StreamId::D2H: return "d2h";
        case StreamId::Host: return "host";
    }
    return "?";
}

const char* op_kind_name(OpKind k) {
    switch (k) {
        case OpKind::WeightXfer: return "WeightXfer";
        case OpKind::Forward: return "Forward";
        case OpKind::Recompute: return "Recompute";
        case OpKind::LocalBackward: return "LocalBackward";
        case OpKind::GradXfer: return "GradXfer";
        case OpKind::Accum: return "Accum";
        case OpKind::OptStep: return "OptStep";
    }
    return "?";
}

std::string trace_to_jsonl(const EventTrace& t) {
    std::ostringstream o;
    o << "{\"meta\":{\"n_layers\":" << t.meta.n_layers << ",\"n_buffers\":" << t.meta.n_buffers
      << ",\"n_slabs\":" << t.meta.n_slabs << ",\"embed_tile\":" << t.meta.embed_tile
      << ",\"head_tile\":" << t.meta.head_tile << "}}\n";
    char buf[128];
    for (const auto& op : t.ops) {
        o << "{\"id\":" << op.id << ",\"stream\":\"" << stream_name(op.stream) << "\",\"kind\":\""
          << op_kind_name(op.kind) << "\",\"layer\":" << op.layer << ",\"buf\":" << op.buf << ",\"slab\":" << op.slab
          << ",\"bytes\":" << op.bytes << ",\"flops\":" << op.flops << ",\"params\":" << op.params
          << ",\"pinned\":" << (op.pinned ? "true" : "false") << ",\"deps\":[";
        for (size_t i = 0; i < op.deps.size(); ++i) o << (i ? "," : "") << op.deps[i];
        std::snprintf(buf, sizeof buf, "],\"t_start_us\":%.3f,\"t_end_us\":%.3f}\n", op.t_start_us, op.t_end_us);
        o << buf;
    }
    return o.str();
}

}  // inline namespace b200
}  // namespace hlm
