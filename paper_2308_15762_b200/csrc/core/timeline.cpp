// Gantt renderings of a SimTrace (ref src/gantt.cpp:25-95, include
// wavepipe/gantt.hpp:32): the same `trace_to_gantt(trace, "svg" | "csv")`
// entry, applicable unchanged to the abstract-time traces of simulate() and
// to the measured traces of the GPU runtime (seconds).  CSV columns match the
// reference's (device,kind,microbatch,slice,start,end); the SVG draws one row
// per device with forward / backward bars coloured by wave direction.
#include <sstream>
#include <stdexcept>

#include "wavepipe/core.hpp"

namespace wavepipe {

namespace {

const char* bar_fill(const TraceInterval& iv) {
  const bool up = iv.direction == Direction::Up;
  switch (iv.kind) {
    case ActionKind::Forward: return up ? "#2196f3" : "#4caf50";
    case ActionKind::Backward: return up ? "#ffeb3b" : "#ff9800";
    default: return "#9c27b0";  // exchanges (abstract time only)
  }
}

std::string timeline_csv(const SimTrace& tr) {
  std::ostringstream out;
  out << "device,kind,microbatch,slice,start,end\n";
  for (size_t dev = 0; dev < tr.intervals.size(); ++dev)
    for (const TraceInterval& iv : tr.intervals[dev])
      out << dev << ',' << action_kind_name(iv.kind) << ',' << iv.microbatch << ',' << iv.slice_index << ','
          << iv.start << ',' << iv.end << '\n';
  return out.str();
}

std::string timeline_svg(const SimTrace& tr) {
  const int rows = static_cast<int>(tr.intervals.size());
  const double x0 = 44.0, y0 = 10.0, pitch = 36.0, bar = 28.0, span_px = 920.0;
  const double scale = span_px / (tr.makespan > 0.0 ? tr.makespan : 1.0);
  std::ostringstream out;
  out << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << x0 + span_px + 10.0 << "\" height=\""
      << y0 + pitch * rows + 24.0 << "\" font-family=\"sans-serif\">\n";
  for (int dev = 0; dev < rows; ++dev) {
    const double y = y0 + dev * pitch;
    out << "  <text x=\"4\" y=\"" << y + bar * 0.7 << "\" font-size=\"12\">d" << dev << "</text>\n"
        << "  <line x1=\"" << x0 << "\" y1=\"" << y + pitch - 4 << "\" x2=\"" << x0 + span_px << "\" y2=\""
        << y + pitch - 4 << "\" stroke=\"#ddd\"/>\n";
    for (const TraceInterval& iv : tr.intervals[dev]) {
      const double x = x0 + iv.start * scale;
      const double w = std::max(0.5, (iv.end - iv.start) * scale);
      out << "  <rect x=\"" << x << "\" y=\"" << y << "\" width=\"" << w << "\" height=\"" << bar << "\" fill=\""
          << bar_fill(iv) << "\" stroke=\"#333\" stroke-width=\"0.5\"/>\n";
      if (iv.kind != ActionKind::BatchedExchange && w >= 9.0)
        out << "  <text x=\"" << x + w / 2 << "\" y=\"" << y + bar * 0.7
            << "\" font-size=\"11\" text-anchor=\"middle\">" << iv.microbatch << "</text>\n";
    }
  }
  const double axis = y0 + pitch * rows + 12.0;
  out << "  <text x=\"" << x0 << "\" y=\"" << axis << "\" font-size=\"11\">0</text>\n"
      << "  <text x=\"" << x0 + span_px << "\" y=\"" << axis << "\" font-size=\"11\" text-anchor=\"end\">"
      << tr.makespan << "</text>\n</svg>\n";
  return out.str();
}

}  // namespace

std::string trace_to_gantt(const SimTrace& trace, const std::string& format) {
  if (format == "csv") return timeline_csv(trace);
  if (format == "svg") return timeline_svg(trace);
  throw std::invalid_argument("unknown gantt format: " + format);
}

}  // namespace wavepipe
