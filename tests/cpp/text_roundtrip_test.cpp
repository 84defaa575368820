// text_roundtrip_test.cpp -- the product's step graphs in the reference's text
// IR format (text.hpp) through host/text_ext.hpp: print -> parse -> print is
// byte-identical, the reparsed function is structurally equal (ir.hpp:686) and
// every let's re-inferred type equals the builder's.
#include <cstdio>

#include "models.hpp"
#include "text_ext.hpp"

using namespace tb;

int main() {
  ensure_registered({});
  int fails = 0;
  for (const char* cfg : {"kind=bert;L=2;H=128;A=2;F=512;V=1024;S=128;B=8;dtype=f32;opt=sgd",
                          "kind=bert;L=2;H=128;A=2;F=512;V=1024;S=128;B=8;dtype=bf16;opt=adam",
                          "kind=gpt2;L=2;H=128;A=2;F=512;V=1024;S=128;B=4;dtype=bf16;opt=adam"}) {
    auto ts = build_train_step(parse_cfg(cfg));
    const std::string a = print_text_ext(*ts.fn);
    ir::ModuleIR back = parse_text_ext(a);
    const auto& fn2 = back.functions.at(0).second;
    const std::string b = print_text_ext(*fn2);
    ir::ModuleIR m;
    m.functions.push_back({back.functions.at(0).first, ts.fn});
    m.entry = back.entry;
    const bool same = a == b, eq = ir::structural_equal(m, back);
    auto s1 = ir::flatten(*ts.fn), s2 = ir::flatten(*fn2);
    int bad_types = 0;
    for (size_t i = 0; i < s1.lets.size() && i < s2.lets.size(); ++i)
      if (!(s1.lets[i].var->ty == s2.lets[i].var->ty)) ++bad_types;
    const bool n_ok = s1.lets.size() == s2.lets.size();
    const bool has_ext = a.substr(0, a.find('\n')).find("i32[") != std::string::npos;
    std::printf("%s: %zu bytes, reprint %s, structural_equal %s, let types %d/%zu differ, i32 header %s\n", cfg,
                a.size(), same ? "identical" : "DIFFERS", eq ? "yes" : "NO", bad_types, s1.lets.size(),
                has_ext ? "yes" : "no");
    fails += !same + !eq + (bad_types != 0) + !n_ok + !has_ext;
  }
  std::printf(fails ? "FAILED\n" : "OK\n");
  return fails ? 1 : 0;
}
