// Mesh and field I/O for the djg command-line tool.
//
//   text mesh   the reference format (mesh.hpp:105-185: "djtled-mesh 1",
//               "nodes N", N coordinate lines, "elements T4|H8 M", M lines of
//               zero-based indices; '#' comment lines), parsed into Real
//   binary mesh "DJGMESH1" + int32 kind, int32 real bytes, int64 N, int64 E,
//               3N Reals, npe*E int32 -- for meshes where text parsing would
//               dominate (50M elements)
//   field       legacy ASCII VTK exactly as export_field (mesh.hpp:266-296),
//               or a NumPy .npy (N x 3 Real) when the path ends in ".npy"
#pragma once

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "config.hpp"

namespace djg::cli {

inline bool ends_with(const std::string& s, const std::string& suffix) {
    return s.size() >= suffix.size() && s.compare(s.size() - suffix.size(), suffix.size(), suffix) == 0;
}

// Reader of the reference's text mesh format (the format and its error
// messages, mesh.hpp:105-185, are the interface): a record cursor that yields
// the significant lines ('#' comment lines and blank lines skipped) with
// their line numbers, and a scanner that reads whitespace-separated fields
// off a record left to right -- a field ends where its number does, so
// "1.5abc" reads 1.5 and leaves "abc" for the next field, like stream
// extraction.
class MeshRecords {
public:
    explicit MeshRecords(std::istream& in) : in_(in) {}

    // Next significant line; ParseError at end of file.
    const std::string& next(const char* expected) {
        while (std::getline(in_, text_)) {
            ++line_;
            const size_t first = text_.find_first_not_of(" \t\r\n\v\f");
            if (first != std::string::npos && text_[first] != '#') {
                pos_ = 0;
                return text_;
            }
        }
        throw ParseError(std::string("unexpected end of file, expected ") + expected, line_);
    }
    long line() const { return line_; }

    bool word(std::string& out) {
        skip_blanks();
        const size_t b = pos_;
        while (pos_ < text_.size() && !std::isspace(static_cast<unsigned char>(text_[pos_]))) ++pos_;
        out.assign(text_, b, pos_ - b);
        return pos_ > b;
    }
    bool integer(long& out) {
        skip_blanks();
        const size_t n = number_prefix(text_.substr(pos_), true);
        if (n == 0) return false;
        out = std::strtol(text_.c_str() + pos_, nullptr, 10);
        pos_ += n;
        return true;
    }
    template <class Real>
    bool real(Real& out) {
        skip_blanks();
        const size_t n = number_prefix(text_.substr(pos_), false);
        if (n == 0 || !convert(text_.substr(pos_, n), out)) return false;
        pos_ += n;
        return true;
    }

private:
    void skip_blanks() {
        while (pos_ < text_.size() && std::isspace(static_cast<unsigned char>(text_[pos_]))) ++pos_;
    }
    std::istream& in_;
    std::string text_;
    size_t pos_ = 0;
    long line_ = 0;
};

template <class Real>
inline Mesh<Real> load_text_mesh(std::istream& in) {
    MeshRecords r(in);
    std::string w;
    long count = 0;
    r.next("header");
    if (!r.word(w) || w != "djtled-mesh" || !r.integer(count)) throw ParseError("expected header 'djtled-mesh 1'", r.line());
    if (count != 1) throw ParseError("unsupported mesh format version " + std::to_string(count), r.line());

    r.next("'nodes N'");
    if (!r.word(w) || w != "nodes" || !r.integer(count) || count < 0) throw ParseError("expected 'nodes N'", r.line());
    Mesh<Real> m;
    m.nodes.resize(size_t(3 * count));
    for (Real* x = m.nodes.data(); x != m.nodes.data() + m.nodes.size(); x += 3) {
        r.next("node coordinates");
        if (!(r.real(x[0]) && r.real(x[1]) && r.real(x[2]))) throw ParseError("malformed node coordinates", r.line());
    }

    r.next("'elements T4|H8 M'");
    std::string kind;
    if (!r.word(w) || w != "elements" || !r.word(kind) || !r.integer(count) || count < 0)
        throw ParseError("expected 'elements T4|H8 M'", r.line());
    if (kind != "T4" && kind != "H8") throw ParseError("unknown element kind '" + kind + "'", r.line());
    m.kind = kind == "T4" ? DJG_T4 : DJG_H8;
    const int npe = m.npe();
    m.conn.resize(size_t(count) * size_t(npe));
    for (int32_t* c = m.conn.data(); c != m.conn.data() + m.conn.size(); c += npe) {
        r.next("element connectivity");
        for (int a = 0; a < npe; ++a) {
            long id;
            if (!r.integer(id)) throw ParseError("expected " + std::to_string(npe) + " node indices", r.line());
            c[a] = int32_t(id);
        }
        long surplus;
        if (r.integer(surplus)) throw ParseError("too many node indices on element line", r.line());
    }
    return m;
}

constexpr char kBinMagic[8] = {'D', 'J', 'G', 'M', 'E', 'S', 'H', '1'};

template <class Real>
inline Mesh<Real> load_binary_mesh(std::istream& in) {
    char magic[8];
    int32_t kind = 0, rb = 0;
    int64_t n = 0, e = 0;
    in.read(magic, 8);
    in.read(reinterpret_cast<char*>(&kind), 4);
    in.read(reinterpret_cast<char*>(&rb), 4);
    in.read(reinterpret_cast<char*>(&n), 8);
    in.read(reinterpret_cast<char*>(&e), 8);
    if (!in || std::memcmp(magic, kBinMagic, 8) != 0) throw ParseError("expected binary mesh header 'DJGMESH1'", 1);
    if ((kind != DJG_T4 && kind != DJG_H8) || (rb != 4 && rb != 8) || n < 0 || e < 0)
        throw ParseError("corrupt binary mesh header", 1);
    Mesh<Real> m;
    m.kind = kind;
    m.nodes.resize(size_t(3 * n));
    if (rb == int32_t(sizeof(Real))) {
        in.read(reinterpret_cast<char*>(m.nodes.data()), std::streamsize(m.nodes.size() * sizeof(Real)));
    } else if (rb == 4) {
        std::vector<float> t(m.nodes.size());
        in.read(reinterpret_cast<char*>(t.data()), std::streamsize(t.size() * 4));
        for (size_t i = 0; i < t.size(); ++i) m.nodes[i] = Real(t[i]);
    } else {
        std::vector<double> t(m.nodes.size());
        in.read(reinterpret_cast<char*>(t.data()), std::streamsize(t.size() * 8));
        for (size_t i = 0; i < t.size(); ++i) m.nodes[i] = Real(t[i]);
    }
    m.conn.resize(size_t(e) * size_t(m.npe()));
    in.read(reinterpret_cast<char*>(m.conn.data()), std::streamsize(m.conn.size() * 4));
    if (!in) throw ParseError("binary mesh is truncated", 1);
    return m;
}

// build_mesh (config.hpp:470-481): generated box or a mesh file relative to
// the config's directory; text or binary by content.
template <class Real>
inline Mesh<Real> build_mesh(const RunConfig<Real>& cfg, const std::string& base_dir) {
    Mesh<Real> m;
    if (cfg.mesh_file.empty()) {
        const double ex[3] = {double(cfg.extent[0]), double(cfg.extent[1]), double(cfg.extent[2])};
        m = generate_box<Real>(ex, cfg.divisions, cfg.kind);
    } else {
        const std::string path = (!base_dir.empty() && cfg.mesh_file.front() != '/') ? base_dir + "/" + cfg.mesh_file
                                                                                    : cfg.mesh_file;
        std::ifstream in(path, std::ios::binary);
        if (!in) throw ConfigError("cannot open mesh file '" + path + "'");
        char head[8] = {};
        in.read(head, 8);
        in.clear();
        in.seekg(0);
        m = std::memcmp(head, kBinMagic, 8) == 0 ? load_binary_mesh<Real>(in) : load_text_mesh<Real>(in);
    }
    validate_mesh(m);
    return m;
}

template <class Real>
inline void save_binary_mesh(const Mesh<Real>& m, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw ConfigError("cannot open output file '" + path + "'");
    const int32_t kind = m.kind, rb = int32_t(sizeof(Real));
    const int64_t n = m.num_nodes(), e = m.num_elements();
    out.write(kBinMagic, 8);
    out.write(reinterpret_cast<const char*>(&kind), 4);
    out.write(reinterpret_cast<const char*>(&rb), 4);
    out.write(reinterpret_cast<const char*>(&n), 8);
    out.write(reinterpret_cast<const char*>(&e), 8);
    out.write(reinterpret_cast<const char*>(m.nodes.data()), std::streamsize(m.nodes.size() * sizeof(Real)));
    out.write(reinterpret_cast<const char*>(m.conn.data()), std::streamsize(m.conn.size() * 4));
}

// render_mesh (mesh.hpp:187-204): full precision, round-trips bit for bit.
template <class Real>
inline void save_text_mesh(const Mesh<Real>& m, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw ConfigError("cannot open output file '" + path + "'");
    out << std::setprecision(std::numeric_limits<Real>::max_digits10);
    out << "djtled-mesh 1\nnodes " << m.num_nodes() << "\n";
    for (int64_t n = 0; n < m.num_nodes(); ++n)
        out << m.nodes[size_t(3 * n)] << " " << m.nodes[size_t(3 * n + 1)] << " " << m.nodes[size_t(3 * n + 2)] << "\n";
    out << "elements " << kind_name(m.kind) << " " << m.num_elements() << "\n";
    const int npe = m.npe();
    for (int64_t e = 0; e < m.num_elements(); ++e)
        for (int a = 0; a < npe; ++a) out << m.conn[size_t(e * npe + a)] << (a + 1 == npe ? "\n" : " ");
}

// export_field (mesh.hpp:266-296) byte for byte, or .npy.
template <class Real>
inline void write_field(const std::string& path, const Mesh<Real>& m, const std::vector<Real>& u) {
    if (int64_t(u.size()) != 3 * m.num_nodes())
        throw ConfigError("displacement count (" + std::to_string(u.size() / 3) + ") does not match node count (" +
                          std::to_string(m.num_nodes()) + ")");
    if (ends_with(path, ".npy")) {
        std::ofstream out(path, std::ios::binary);
        if (!out) throw ConfigError("cannot open output file '" + path + "'");
        std::string hdr = std::string("{'descr': '<") + (sizeof(Real) == 4 ? "f4" : "f8") +
                          "', 'fortran_order': False, 'shape': (" + std::to_string(m.num_nodes()) + ", 3), }";
        while ((10 + hdr.size() + 1) % 64 != 0) hdr += ' ';
        hdr += '\n';
        const uint16_t hl = uint16_t(hdr.size());
        out.write("\x93NUMPY\x01\x00", 8);
        out.write(reinterpret_cast<const char*>(&hl), 2);
        out << hdr;
        out.write(reinterpret_cast<const char*>(u.data()), std::streamsize(u.size() * sizeof(Real)));
        return;
    }
    std::ofstream out(path);
    if (!out) throw ConfigError("cannot open output file '" + path + "'");
    const char* scalar = sizeof(Real) == 4 ? "float" : "double";
    const int npe = m.npe();
    const int64_t N = m.num_nodes(), E = m.num_elements();
    std::ostringstream o;
    o << std::setprecision(std::numeric_limits<Real>::max_digits10);
    o << "# vtk DataFile Version 3.0\ndjtled displacement field\nASCII\nDATASET UNSTRUCTURED_GRID\n";
    o << "POINTS " << N << " " << scalar << "\n";
    for (int64_t n = 0; n < N; ++n)
        o << m.nodes[size_t(3 * n)] << " " << m.nodes[size_t(3 * n + 1)] << " " << m.nodes[size_t(3 * n + 2)] << "\n";
    o << "CELLS " << E << " " << E * (npe + 1) << "\n";
    for (int64_t e = 0; e < E; ++e) {
        o << npe;
        for (int a = 0; a < npe; ++a) o << " " << m.conn[size_t(e * npe + a)];
        o << "\n";
    }
    o << "CELL_TYPES " << E << "\n";
    const int cell_type = m.kind == DJG_T4 ? 10 : 12;
    for (int64_t e = 0; e < E; ++e) o << cell_type << "\n";
    o << "POINT_DATA " << N << "\n";
    o << "VECTORS displacement " << scalar << "\n";
    for (int64_t n = 0; n < N; ++n) o << u[size_t(3 * n)] << " " << u[size_t(3 * n + 1)] << " " << u[size_t(3 * n + 2)] << "\n";
    out << o.str();
}

}  // namespace djg::cli
