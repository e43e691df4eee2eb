// ORACLE BUILD SHIM — TEST INFRASTRUCTURE ONLY. nlohmann/json is vendored by
// the reference under proj/vendor/, which its .gitignore leaves out
// (proj/.gitignore:2), so it is absent here. This is a small JSON value type
// with the part of nlohmann::json's API the reference's core sources call
// (geometry.cpp:142-240, io.cpp:18-213, simulator.cpp:185-240,
// trainer.cpp:38-131): parse / dump, operator[] (auto-vivifying objects),
// at / value / contains / size / is_array, get<T>, key()/value() iteration and
// nlohmann's initializer-list rule (a list whose elements are all [string, x]
// pairs is an object, anything else an array). Objects keep keys sorted
// (nlohmann::json's default std::map). Numbers dump as integers when they were
// stored as integers, otherwise as the shortest round-trip decimal.
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <istream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace nlohmann {

class json {
 public:
  enum class kind { null, boolean, integer, unsigned_integer, floating, string, array, object };

  struct exception : std::runtime_error {
    using std::runtime_error::runtime_error;
  };
  struct parse_error : exception {
    using exception::exception;
  };
  struct type_error : exception {
    using exception::exception;
  };
  struct out_of_range : exception {
    using exception::exception;
  };

  json() = default;
  json(std::nullptr_t) {}
  json(bool b) : k_(kind::boolean), b_(b) {}
  template <typename T, std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, bool> &&
                                             std::is_signed_v<T>, int> = 0>
  json(T v) : k_(kind::integer), i_(static_cast<int64_t>(v)) {}
  template <typename T, std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, bool> &&
                                             std::is_unsigned_v<T>, int> = 0>
  json(T v) : k_(kind::unsigned_integer), u_(static_cast<uint64_t>(v)) {}
  json(double v) : k_(kind::floating), d_(v) {}
  json(float v) : k_(kind::floating), d_(v) {}
  json(const char* s) : k_(kind::string), s_(s) {}
  json(const std::string& s) : k_(kind::string), s_(s) {}
  template <typename T>
  json(const std::vector<T>& v) : k_(kind::array) {
    for (const auto& x : v) a_.emplace_back(x);
  }
  json(std::initializer_list<json> init) {
    bool is_object = init.size() > 0;
    for (const auto& e : init)
      if (!(e.k_ == kind::array && e.a_.size() == 2 && e.a_[0].k_ == kind::string)) is_object = false;
    if (is_object) {
      k_ = kind::object;
      for (const auto& e : init) o_[e.a_[0].s_] = e.a_[1];
    } else {
      k_ = kind::array;
      a_.assign(init.begin(), init.end());
    }
  }
  static json array(std::initializer_list<json> init = {}) {
    json j;
    j.k_ = kind::array;
    j.a_.assign(init.begin(), init.end());
    return j;
  }
  static json object() {
    json j;
    j.k_ = kind::object;
    return j;
  }

  // ---- queries
  bool is_null() const { return k_ == kind::null; }
  bool is_array() const { return k_ == kind::array; }
  bool is_object() const { return k_ == kind::object; }
  bool is_string() const { return k_ == kind::string; }
  bool is_number() const {
    return k_ == kind::integer || k_ == kind::unsigned_integer || k_ == kind::floating;
  }
  size_t size() const {
    if (k_ == kind::array) return a_.size();
    if (k_ == kind::object) return o_.size();
    return k_ == kind::null ? 0 : 1;
  }
  bool contains(const std::string& key) const { return k_ == kind::object && o_.count(key) > 0; }

  // ---- element access
  json& operator[](const std::string& key) {
    if (k_ == kind::null) k_ = kind::object;
    if (k_ != kind::object) throw type_error("operator[] with a key on a non-object");
    return o_[key];
  }
  json& operator[](const char* key) { return (*this)[std::string(key)]; }
  const json& operator[](const std::string& key) const { return at(key); }
  const json& operator[](const char* key) const { return at(std::string(key)); }
  json& operator[](size_t i) {
    if (k_ == kind::null) k_ = kind::array;
    if (k_ != kind::array) throw type_error("operator[] with an index on a non-array");
    if (i >= a_.size()) a_.resize(i + 1);
    return a_[i];
  }
  const json& operator[](size_t i) const { return at(i); }
  json& operator[](int i) { return (*this)[static_cast<size_t>(i)]; }
  const json& operator[](int i) const { return at(static_cast<size_t>(i)); }

  const json& at(const std::string& key) const {
    if (k_ != kind::object) throw type_error("at(key) on a non-object");
    auto it = o_.find(key);
    if (it == o_.end()) throw out_of_range("key '" + key + "' not found");
    return it->second;
  }
  const json& at(const char* key) const { return at(std::string(key)); }
  const json& at(size_t i) const {
    if (k_ != kind::array) throw type_error("at(index) on a non-array");
    if (i >= a_.size()) throw out_of_range("array index out of range");
    return a_[i];
  }
  const json& at(int i) const { return at(static_cast<size_t>(i)); }

  std::string value(const std::string& key, const char* def) const {
    if (!contains(key)) return def;
    return at(key).get<std::string>();
  }
  template <typename T>
  T value(const std::string& key, T def) const {
    if (!contains(key)) return def;
    return at(key).get<T>();
  }

  // ---- conversion
  template <typename T>
  T get() const {
    if constexpr (std::is_same_v<T, bool>) {
      if (k_ != kind::boolean) throw type_error("type must be boolean");
      return b_;
    } else if constexpr (std::is_integral_v<T> || std::is_floating_point_v<T>) {
      switch (k_) {
        case kind::integer: return static_cast<T>(i_);
        case kind::unsigned_integer: return static_cast<T>(u_);
        case kind::floating: return static_cast<T>(d_);
        default: throw type_error("type must be number");
      }
    } else if constexpr (std::is_same_v<T, std::string>) {
      if (k_ != kind::string) throw type_error("type must be string");
      return s_;
    } else if constexpr (std::is_same_v<T, json>) {
      return *this;
    } else {
      if (k_ != kind::array) throw type_error("type must be array");
      T out;
      for (const auto& e : a_) out.push_back(e.template get<typename T::value_type>());
      return out;
    }
  }

  // ---- iteration (arrays yield elements, objects yield values with key())
  class const_iterator {
   public:
    const json* j;
    size_t ai;
    std::map<std::string, json>::const_iterator oi;
    const json& operator*() const { return j->k_ == kind::object ? oi->second : j->a_[ai]; }
    const json* operator->() const { return &**this; }
    const_iterator& operator++() {
      if (j->k_ == kind::object) ++oi;
      else ++ai;
      return *this;
    }
    bool operator==(const const_iterator& o) const {
      return j->k_ == kind::object ? oi == o.oi : ai == o.ai;
    }
    bool operator!=(const const_iterator& o) const { return !(*this == o); }
    const std::string& key() const {
      if (j->k_ != kind::object) throw type_error("key() on a non-object iterator");
      return oi->first;
    }
    const json& value() const { return **this; }
  };
  const_iterator begin() const {
    return const_iterator{this, 0, o_.begin()};
  }
  const_iterator end() const {
    return const_iterator{this, k_ == kind::array ? a_.size() : 0, o_.end()};
  }

  // ---- serialisation
  std::string dump(int indent = -1) const {
    std::string out;
    dump_to(out, indent, 0);
    return out;
  }

  static json parse(const std::string& text) {
    size_t p = 0;
    json j = parse_value(text, p);
    skip_ws(text, p);
    if (p != text.size()) throw parse_error("syntax error: trailing characters");
    return j;
  }
  friend std::istream& operator>>(std::istream& in, json& j) {
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    j = parse(text);
    return in;
  }

 private:
  kind k_ = kind::null;
  bool b_ = false;
  int64_t i_ = 0;
  uint64_t u_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<json> a_;
  std::map<std::string, json> o_;

  static void dump_string(std::string& out, const std::string& s) {
    out += '"';
    for (char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\n': out += "\\n"; break;
        case '\t': out += "\\t"; break;
        case '\r': out += "\\r"; break;
        default: out += c;
      }
    }
    out += '"';
  }
  void dump_to(std::string& out, int indent, int level) const {
    auto nl = [&](int lv) {
      if (indent < 0) return;
      out += '\n';
      out.append(static_cast<size_t>(indent * lv), ' ');
    };
    switch (k_) {
      case kind::null: out += "null"; break;
      case kind::boolean: out += b_ ? "true" : "false"; break;
      case kind::integer: out += std::to_string(i_); break;
      case kind::unsigned_integer: out += std::to_string(u_); break;
      case kind::floating: {
        if (!std::isfinite(d_)) {
          out += "null";
          break;
        }
        char buf[64];
        // nlohmann prints decimal notation for moderate magnitudes, else an exponent
        const double ad = std::fabs(d_);
        const bool fixed = ad == 0.0 || (ad >= 1e-4 && ad < 1e15);
        auto r = fixed ? std::to_chars(buf, buf + sizeof(buf), d_, std::chars_format::fixed)
                       : std::to_chars(buf, buf + sizeof(buf), d_, std::chars_format::scientific);
        std::string s(buf, r.ptr);
        if (s.find_first_of(".eE") == std::string::npos) s += ".0";
        out += s;
        break;
      }
      case kind::string: dump_string(out, s_); break;
      case kind::array: {
        out += '[';
        for (size_t i = 0; i < a_.size(); ++i) {
          if (i) out += ',';
          nl(level + 1);
          a_[i].dump_to(out, indent, level + 1);
        }
        if (!a_.empty()) nl(level);
        out += ']';
        break;
      }
      case kind::object: {
        out += '{';
        bool first = true;
        for (const auto& [key, v] : o_) {
          if (!first) out += ',';
          first = false;
          nl(level + 1);
          dump_string(out, key);
          out += indent < 0 ? ":" : ": ";
          v.dump_to(out, indent, level + 1);
        }
        if (!o_.empty()) nl(level);
        out += '}';
        break;
      }
    }
  }

  static void skip_ws(const std::string& t, size_t& p) {
    while (p < t.size() && (t[p] == ' ' || t[p] == '\n' || t[p] == '\r' || t[p] == '\t')) ++p;
  }
  static json parse_value(const std::string& t, size_t& p) {
    skip_ws(t, p);
    if (p >= t.size()) throw parse_error("syntax error: unexpected end of input");
    const char c = t[p];
    if (c == '{') {
      ++p;
      json j = object();
      skip_ws(t, p);
      if (p < t.size() && t[p] == '}') {
        ++p;
        return j;
      }
      while (true) {
        skip_ws(t, p);
        if (p >= t.size() || t[p] != '"') throw parse_error("syntax error: expected a key");
        const std::string key = parse_string(t, p);
        skip_ws(t, p);
        if (p >= t.size() || t[p] != ':') throw parse_error("syntax error: expected ':'");
        ++p;
        j.o_[key] = parse_value(t, p);
        skip_ws(t, p);
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == '}') {
          ++p;
          return j;
        }
        throw parse_error("syntax error: expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p;
      json j = array();
      skip_ws(t, p);
      if (p < t.size() && t[p] == ']') {
        ++p;
        return j;
      }
      while (true) {
        j.a_.push_back(parse_value(t, p));
        skip_ws(t, p);
        if (p < t.size() && t[p] == ',') {
          ++p;
          continue;
        }
        if (p < t.size() && t[p] == ']') {
          ++p;
          return j;
        }
        throw parse_error("syntax error: expected ',' or ']'");
      }
    }
    if (c == '"') return json(parse_string(t, p));
    if (t.compare(p, 4, "true") == 0) {
      p += 4;
      return json(true);
    }
    if (t.compare(p, 5, "false") == 0) {
      p += 5;
      return json(false);
    }
    if (t.compare(p, 4, "null") == 0) {
      p += 4;
      return json();
    }
    const size_t start = p;
    bool is_float = false;
    if (p < t.size() && (t[p] == '-' || t[p] == '+')) ++p;
    while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '.' ||
                            t[p] == 'e' || t[p] == 'E' || t[p] == '-' || t[p] == '+')) {
      if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') is_float = true;
      ++p;
    }
    if (p == start) throw parse_error("syntax error: invalid literal");
    const std::string num = t.substr(start, p - start);
    try {
      if (!is_float) {
        if (num[0] == '-') return json(static_cast<int64_t>(std::stoll(num)));
        return json(static_cast<uint64_t>(std::stoull(num)));
      }
      return json(std::stod(num));
    } catch (const std::exception&) {
      throw parse_error("syntax error: bad number '" + num + "'");
    }
  }
  static std::string parse_string(const std::string& t, size_t& p) {
    ++p;  // opening quote
    std::string s;
    while (p < t.size() && t[p] != '"') {
      if (t[p] == '\\' && p + 1 < t.size()) {
        ++p;
        switch (t[p]) {
          case 'n': s += '\n'; break;
          case 't': s += '\t'; break;
          case 'r': s += '\r'; break;
          default: s += t[p];
        }
      } else {
        s += t[p];
      }
      ++p;
    }
    if (p >= t.size()) throw parse_error("syntax error: unterminated string");
    ++p;
    return s;
  }
};

}  // namespace nlohmann
